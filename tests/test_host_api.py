"""CPU tests of the host-side mirror of the reference API (no GPU needed):
config validation, the prune rule, boost tables, streaming value objects,
graph text I/O and FlatGraph construction -- mirroring the reference's
test_decoder.py / test_boosting.py / test_streaming.py / test_wfst.py cases
for these names."""

import math

import numpy as np
import pytest

import paper_2311_04996_b200 as P
from paper_2311_04996_b200 import errors
from paper_2311_04996_b200.wfst import Arc, SymbolTable, Wfst, arc_sort, read_fst_text, read_symbols, write_fst_text


def test_decoder_config_validation():
    P.DecoderConfig()
    for bad in (dict(beam=0), dict(beam=-1.0), dict(max_active=0), dict(acoustic_scale=0.0)):
        with pytest.raises(ValueError):
            P.DecoderConfig(**bad)
    assert P.DecoderConfig().beam == 17.0 and P.DecoderConfig().max_active == 10_000


def test_prune_rule_beam_then_max_active_by_cost_state():
    T = P.Token
    toks = [T(0, 1.0, -1), T(1, 5.0, -1), T(2, 20.0, -1)]
    assert [t.state for t in P.prune(toks, 10.0, 10)] == [0, 1]
    tied = [T(5, 1.0, -1), T(3, 1.0, -1), T(9, 0.5, -1)]
    assert [t.state for t in P.prune(tied, 100.0, 2)] == [3, 9]  # (cost, state) ranking, state order out
    with pytest.raises(ValueError):
        P.prune([], 1.0, 1)


def test_boost_table_parse_and_dense_costs():
    words = SymbolTable()
    for w in ("alpha", "beta", "gamma"):
        words.add(w)
    tab, skipped = P.load_boost_table("alpha 2.5\n\nzeta 1\nbeta\t0.5\n", words)
    assert skipped == ["zeta"]
    assert tab.entries == {1: -2.5, 2: -0.5}
    v = P.boost_costs(tab, 3)
    assert v.dtype == np.float64 and v.tolist() == [0.0, -2.5, -0.5, 0.0]
    assert P.boost_costs(P.BoostTable(), 3) is None  # empty table -> unboosted path
    with pytest.raises(errors.BoostError):
        P.BoostTable(entries={0: -1.0})
    with pytest.raises(errors.BoostParseError, match="line 1"):
        P.load_boost_table("alpha x\n", words)
    fsa = P.build_boost_fsa(tab, words)
    assert fsa.num_states == 1 and {a.ilabel: a.weight for a in fsa.arcs(0)} == {1: -2.5, 2: -0.5, 3: 0.0}


def test_stream_value_objects():
    with pytest.raises(P.StreamError, match="final"):
        P.Chunk(stream_id=0, frames=np.zeros((0, 3)))
    P.Chunk(stream_id=0, frames=np.zeros((0, 3)), is_last=True)
    with pytest.raises(P.StreamError):
        P.BatcherConfig(max_batch=0)
    with pytest.raises(P.StreamError):
        P.BatcherConfig(max_wait_ms=-1)


def test_fst_text_roundtrip_and_errors():
    g = Wfst(num_states=3, start=1)
    g.add_arc(1, Arc(2, 3, 0.25, 0))
    g.add_arc(0, Arc(0, 0, 1.0, 2))
    g.set_final(2, 0.5)
    txt = write_fst_text(g)
    assert txt.splitlines()[0].startswith("1 0 2 3")
    assert read_fst_text(txt) == g
    with pytest.raises(errors.FstParseError, match="line 1"):
        read_fst_text("0 1 x 2\n")
    with pytest.raises(errors.FstParseError):
        read_fst_text("")
    syms = read_symbols("<eps> 0\na 1\nb 2\n")
    assert syms.id("b") == 2 and syms.symbol(1) == "a" and len(syms) == 3
    with pytest.raises(errors.FstParseError):
        read_symbols("a 1\n")


def test_flatgraph_layout_matches_reference_convention():
    g = Wfst(num_states=3, start=0)
    g.add_arc(0, Arc(2, 5, 0.5, 1))
    g.add_arc(0, Arc(0, 0, 0.1, 2))
    g.add_arc(0, Arc(1, 4, 0.2, 2))
    g.add_arc(2, Arc(0, 7, 0.0, 1))
    g.set_final(1, 0.3)
    fg = P.flatten(g)
    assert fg.off.tolist() == [0, 3, 3, 4]
    assert fg.eps_end.tolist() == [1, 3, 4]
    assert fg.ilabel.tolist() == [0, 1, 2, 0]  # stable sort by ilabel per state
    assert fg.olabel.tolist() == [0, 4, 5, 7]
    assert math.isinf(fg.final[0]) and fg.final[1] == 0.3
    assert (fg.max_ilabel, fg.max_olabel) == (2, 7)
    assert P.flatten(g) is fg  # cached on the Wfst
    with pytest.raises(errors.DecodeError, match="empty"):
        P.flatten(Wfst.empty())


def test_arc_sort_is_stable():
    g = Wfst(num_states=2, start=0)
    for lab, w in ((2, 0.1), (1, 0.2), (2, 0.3)):
        g.add_arc(0, Arc(lab, 0, w, 1))
    assert [a.weight for a in arc_sort(g).arcs(0)] == [0.2, 0.1, 0.3]
    with pytest.raises(ValueError):
        arc_sort(g, "weight")
