"""Generate the golden parity fixtures in tests/golden/ FROM THE REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package straight from
/root/reference/pkg/src (pure-Python kernel: _pykernel.py, bit-identical to the
compiled one per the reference's own test_kernels.py) and the reference test
builders (pkg/tests/conftest.py), decodes a fixed set of cases and stores,
per case, the graph CSR arrays, the log-likelihoods, the decoder config, the
boost vector, and the reference results: per-frame history records
(prev, olabels, state, cost), active tokens, best path, or the error message.
The fixtures are read by tests/test_oracle.py (CPU) and tests/test_gpu_parity.py
(GPU) -- /root/reference is never read at test time.
"""

from __future__ import annotations

import math
import os
import sys
from pathlib import Path

import numpy as np

os.environ["CTCWFST_PURE_PYTHON"] = "1"
sys.path[:0] = ["/root/reference/pkg/src", "/root/reference/pkg/tests"]

from conftest import make_toy_system, planted_frames, random_frames  # noqa: E402
from ctcwfst.boosting import BoostTable, boost_costs  # noqa: E402
from ctcwfst.decoder import DecoderConfig, DecodeState, best_path, flatten  # noqa: E402
from ctcwfst.errors import DecodeError  # noqa: E402
from ctcwfst.wfst import Arc, Wfst, arc_sort  # noqa: E402

OUT = Path(__file__).resolve().parent
WIDE = dict(beam=1e9, max_active=10**9)


def chain_graph():
    """test_decoder.py:28-36"""
    g = Wfst(num_states=4, start=0)
    g.add_arc(0, Arc(1, 1, 0.3, 1))
    g.add_arc(0, Arc(0, 0, 0.0, 3))
    g.add_arc(1, Arc(2, 0, 0.1, 2))
    g.set_final(2, 0.25)
    g.set_final(3, 0.0)
    return arc_sort(g, "ilabel")


def config1_system(seed):
    """BASELINE config 1 with the reference's own builders: 29 chars + blank
    (blank id 0), 50-word lexicon (prons 2-7 chars), random bigram ARPA
    (conftest.random_arpa_text), compact topology, build_tlg."""
    from conftest import random_arpa_text
    from ctcwfst.arpa import build_grammar_fst, parse_arpa
    from ctcwfst.graph import build_tlg
    from ctcwfst.lexicon import LexiconEntry, build_lexicon_fst, word_symbols
    from ctcwfst.topology import UnitInventory, build_ctc_topo_compact
    from ctcwfst.wfst import SymbolTable

    rng = np.random.default_rng(seed)
    units = SymbolTable()
    units.add("<blk>")
    for i in range(29):
        units.add(f"c{i:02d}")
    inv = UnitInventory(units=units, blank_id=0)
    prons = set()
    while len(prons) < 50:
        n = int(rng.integers(2, 8))
        prons.add(tuple(int(rng.integers(1, 30)) for _ in range(n)))
    entries = [LexiconEntry(word="w" + "_".join(map(str, p)), pronunciation=p) for p in sorted(prons)]
    words = word_symbols(entries)
    arpa = random_arpa_text(rng, sorted(e.word for e in entries), 2)
    tlg = build_tlg(build_ctc_topo_compact(inv), build_lexicon_fst(entries, inv, words),
                    build_grammar_fst(parse_arpa(arpa), words))
    return tlg, [e.pronunciation for e in entries]


def c1_frames(rng, prons, V, n_frames, gap=12.0, noise=0.5):
    """conftest.planted_frames rendering (unit repeats + blanks, whole words)."""
    path = []
    while True:
        pron = prons[int(rng.integers(0, len(prons)))]
        r = []
        for u in pron:
            r.extend([u] * int(rng.integers(1, 3)))
            r.append(0)
        if len(path) + len(r) > n_frames:
            break
        path.extend(r)
    path.extend([0] * (n_frames - len(path)))
    mat = rng.normal(-gap, noise, size=(n_frames, V))
    mat[np.arange(n_frames), path] = rng.normal(-0.05, 0.02, size=n_frames)
    return mat


def save(name, graph, chunks, cfg_kw, boost=None, boost_poke=False):
    """Decode `chunks` (list of (F, V) arrays) through one reference channel."""
    fg = flatten(graph)
    cfg = DecoderConfig(**cfg_kw)
    ch = DecodeState(fg, cfg)
    if boost is not None:
        if boost_poke:
            ch.boost = boost  # direct assignment, no re-seed (test_decoder.py:343)
        else:
            ch.set_boost(boost)
    seed_tokens = ch.active_tokens()
    err = ""
    ok_chunks = 0
    for c in chunks:
        try:
            ch.advance_frames(c)
            ok_chunks += 1
        except DecodeError as e:
            err = str(e)
            break
    hist = ch.history_records()
    d = dict(
        num_states=fg.num_states, start=fg.start, off=fg.off, eps_end=fg.eps_end, ilabel=fg.ilabel,
        olabel=fg.olabel, weight=fg.weight, nextstate=fg.nextstate, final=fg.final,
        chunk_sizes=np.asarray([len(c) for c in chunks], np.int64),
        frames=np.concatenate(chunks) if chunks else np.zeros((0, 1)),
        beam=cfg.beam, max_active=cfg.max_active, acoustic_scale=cfg.acoustic_scale,
        relax_eps=cfg.nonemitting_relax_epsilon,
        max_ne_iters=-1 if cfg.max_nonemitting_iters is None else cfg.max_nonemitting_iters,
        boost=np.zeros(0) if boost is None else np.asarray(boost, np.float64),
        has_boost=boost is not None, boost_poke=boost_poke,
        error=err, ok_chunks=ok_chunks,
        seed_state=np.asarray([t.state for t in seed_tokens], np.int32),
        seed_cost=np.asarray([t.cost for t in seed_tokens]),
        seed_chain_off=ch.act_chain_off if ch.frame_count == 0 else np.zeros(0, np.int64),
        seed_chain_pool=ch.act_chain_pool if ch.frame_count == 0 else np.zeros(0, np.int32),
        counts=np.asarray([len(f) for f in hist], np.int64),
        rec_prev=np.asarray([r[0] for f in hist for r in f], np.int64),
        rec_state=np.asarray([r[2] for f in hist for r in f], np.int32),
        rec_cost=np.asarray([r[3] for f in hist for r in f], np.float64),
        rec_olab_len=np.asarray([len(r[1]) for f in hist for r in f], np.int64),
        rec_olab=np.asarray([o for f in hist for r in f for o in r[1]], np.int32),
        tok_state=np.asarray([t.state for t in ch.active_tokens()], np.int32),
        tok_cost=np.asarray([t.cost for t in ch.active_tokens()], np.float64),
        tok_bp=np.asarray([t.backpointer for t in ch.active_tokens()], np.int64),
    )
    if ch.frame_count:
        h = best_path(ch)
        d.update(best_words=np.asarray(h.words, np.int32), best_cost=h.total_cost, frame_count=h.frame_count)
    else:
        d.update(best_words=np.zeros(0, np.int32), best_cost=math.nan, frame_count=0)
    np.savez_compressed(OUT / f"{name}.npz", **d)
    return d


def main():
    for p in OUT.glob("*.npz"):
        p.unlink()
    # -- known-answer cases (test_decoder.py) --
    save("kat_expansion", chain_graph(), [np.array([[-0.2, -5.0]])], WIDE)
    save("kat_scale", chain_graph(), [np.array([[-0.2, -5.0]])], dict(WIDE, acoustic_scale=0.5))
    g = Wfst(num_states=3, start=0)
    g.add_arc(0, Arc(1, 0, 1.1, 2))
    g.add_arc(0, Arc(2, 0, 0.7, 2))
    g.set_final(2)
    save("kat_recombination", arc_sort(g, "ilabel"), [np.array([[0.0, -0.2]])], WIDE)
    save("kat_final_pref", chain_graph(), [np.array([[-0.2, -5.0]]), np.array([[-5.0, -0.2]])], WIDE)
    g = Wfst(num_states=3, start=0)
    g.add_arc(0, Arc(1, 1, 0.0, 1))
    g.add_arc(1, Arc(1, 0, 0.0, 2))
    g.set_final(2)
    save("kat_fallback", arc_sort(g, "ilabel"), [np.array([[-0.5]])], WIDE)
    g = Wfst(num_states=3, start=0)
    g.add_arc(0, Arc(0, 0, 0.1, 1))
    g.add_arc(1, Arc(1, 2, 0.0, 2))
    g.set_final(2)
    save("kat_eps_only", arc_sort(g, "ilabel"), [np.array([[-0.3]])], WIDE)
    g = Wfst(num_states=3, start=0)
    g.add_arc(0, Arc(1, 0, 0.0, 1))
    g.add_arc(1, Arc(0, 1, 0.0, 2))
    g.add_arc(2, Arc(0, 1, 0.0, 1))
    g.set_final(1)
    save("kat_eps_cycle", arc_sort(g, "ilabel"), [np.array([[-0.1]])], WIDE,
         boost=np.array([0.0, -1.0]), boost_poke=True)
    save("kat_dead_beam", chain_graph(), [np.array([[-0.2, -5.0], [-np.inf, -np.inf], [-0.2, -5.0]])], WIDE)
    # epsilon arcs carrying olabels (right-pushed style), exercises chains
    g = Wfst(num_states=5, start=0)
    g.add_arc(0, Arc(0, 7, 0.2, 1))
    g.add_arc(1, Arc(0, 8, 0.1, 2))
    g.add_arc(2, Arc(1, 3, 0.5, 3))
    g.add_arc(3, Arc(0, 9, 0.0, 4))
    g.add_arc(4, Arc(2, 0, 0.0, 4))
    g.add_arc(3, Arc(1, 0, 0.3, 3))
    g.set_final(4)
    g.set_final(3, 1.0)
    save("kat_eps_olabels", arc_sort(g, "ilabel"), [np.array([[-0.1, -2.0], [-3.0, -0.2], [-0.4, -0.1]])], WIDE)
    # -- test_kernels.py-style random systems --
    for seed in range(16):
        sysm = make_toy_system(seed=60 + seed, num_units=2 + seed % 4, num_words=3 + seed % 5,
                               order=1 + seed % 2, compact=seed % 3 != 0)
        rng = np.random.default_rng(200 + seed)
        frames = (planted_frames if seed % 2 else random_frames)(rng, sysm, 15, 45)
        cfg = dict(beam=float(rng.choice([2.0, 6.0, 17.0, 1e9])), max_active=int(rng.choice([3, 17, 10_000])))
        boost = None
        if seed % 3 == 0:
            wid = sysm.words.id(sysm.entries[0].word)
            boost = boost_costs(BoostTable(entries={wid: -4.0}), sysm.words.max_id())
        chunk = [None, 1, 7, 13][seed % 4]
        chunks = [frames] if chunk is None else [frames[i:i + chunk] for i in range(0, len(frames), chunk)]
        save(f"rand_{seed:02d}", sysm.tlg, chunks, cfg, boost)
    # -- config-1-like: V=30 (29 chars + blank), 50 words, bigram, 4 x 200 planted frames --
    tlg, rendered = config1_system(seed=1)
    rng = np.random.default_rng(11)
    for u in range(4):
        frames = c1_frames(rng, rendered, 29 + 1, 200)
        save(f"c1_utt{u}", tlg, [frames], dict(beam=17.0, max_active=10_000))
    print("wrote", len(list(OUT.glob('*.npz'))), "fixtures")


if __name__ == "__main__":
    main()
