"""Binary CSR graph files (graphio.py, ctw_graph_load): round trips and
malformed-file errors on the CPU; decode from a loaded file on the GPU."""

import ctypes as C

import numpy as np
import pytest


def _system():
    from paper_2311_04996_b200 import synth

    return synth.build_system(synth.SystemSpec(num_units=12, num_words=40, order=3, seed=4, min_pron=1, max_pron=4))


def test_roundtrip_arrays(tmp_path):
    from paper_2311_04996_b200 import graphio

    fg = _system().graph
    p = graphio.save_graph(fg, tmp_path / "g.ctwg")
    for mm in (True, False):
        g2 = graphio.load_graph(p, mmap=mm)
        for k in ("off", "eps_end", "ilabel", "olabel", "weight", "nextstate", "final"):
            assert np.array_equal(np.asarray(getattr(g2, k)), getattr(fg, k)), k
        assert (g2.num_states, g2.start, g2.max_ilabel, g2.max_olabel, g2.num_arcs) == \
            (fg.num_states, fg.start, fg.max_ilabel, fg.max_olabel, fg.num_arcs)


def test_bad_files(tmp_path):
    from paper_2311_04996_b200 import GraphError, graphio

    fg = _system().graph
    p = graphio.save_graph(fg, tmp_path / "g.ctwg")
    raw = p.read_bytes()
    (tmp_path / "bad.ctwg").write_bytes(b"NOTGRAPH" + raw[8:])
    with pytest.raises(GraphError, match="not a CTWGRAPH"):
        graphio.load_graph(tmp_path / "bad.ctwg")
    (tmp_path / "short.ctwg").write_bytes(raw[: len(raw) // 2])
    with pytest.raises(GraphError, match="truncated"):
        graphio.load_graph(tmp_path / "short.ctwg")


@pytest.mark.gpu
def test_decode_from_file_and_c_loader(tmp_path):
    from paper_2311_04996_b200 import DecoderConfig, _lib, decode_batch, graphio, synth

    s = _system()
    p = graphio.save_graph(s.graph, tmp_path / "g.ctwg")
    utts = synth.planted_utterances(s, 4, 50, seed=2)
    cfg = DecoderConfig(beam=14.0, max_active=300)
    want = decode_batch(s.graph, cfg, utts)
    got = decode_batch(graphio.load_graph(p), cfg, utts)
    assert got == want
    # the C-ABI loader (no Python in the load path)
    L = _lib.load()
    h = C.c_void_p()
    _lib.check(L.ctw_graph_load(str(p).encode(), 0, C.byref(h)), "graph load")
    v = [C.c_int64() for _ in range(5)]
    L.ctw_graph_info(h, *[C.byref(x) for x in v])
    assert v[0].value == s.graph.num_states and v[1].value == s.graph.num_arcs
    L.ctw_graph_destroy(h)
    assert L.ctw_graph_load(str(tmp_path / "missing.ctwg").encode(), 0, C.byref(h)) != 0
