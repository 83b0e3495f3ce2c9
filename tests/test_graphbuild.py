"""The native graph builder (csrc/ctw_graphbuild.cpp + synth.py) reproduces
the reference's offline construction exactly: T o (L o G) composition,
trim and arc sort state-for-state (reference graph.py:9-17, wfst.py:294-410),
and the ARPA grammar acceptor (arpa.py:140-205). CPU only; uses the compiled
reference in oracle/_ref and the reference's own test builders."""

import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import ref_available

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def _same(a, b):
    return (a.start == b.start and a.num_states == b.num_states and a.finals == b.finals
            and all([tuple(x) for x in a.arcs(s)] == [tuple(x) for x in b.arcs(s)] for s in a.states()))


def _ref_toy(seed, **kw):
    """A toy system built with the reference's own conftest recipe."""
    from ctcwfst.arpa import build_grammar_fst, parse_arpa
    from ctcwfst.graph import build_tlg
    from ctcwfst.lexicon import LexiconEntry, build_lexicon_fst, word_symbols
    from ctcwfst.topology import UnitInventory, build_ctc_topo_compact, build_ctc_topo_normal
    from ctcwfst.wfst import SymbolTable

    rng = np.random.default_rng(seed)
    nu = kw.get("num_units", 3)
    units = SymbolTable()
    units.add("<blk>")
    for c in "abcde"[:nu]:
        units.add(c)
    inv = UnitInventory(units=units, blank_id=0)
    prons = set()
    while len(prons) < kw.get("num_words", 5):
        prons.add(tuple(int(rng.integers(1, nu + 1)) for _ in range(int(rng.integers(1, 4)))))
    entries = [LexiconEntry(word="".join("abcde"[u - 1] for u in p) + "_w", pronunciation=p) for p in sorted(prons)]
    words = word_symbols(entries)
    vocab = sorted(e.word for e in entries)
    lines = ["\\data\\", f"ngram 1={len(vocab) + 2}", "", "\\1-grams:", "-99\t<s>", "-1.0\t</s>"]
    lp = rng.dirichlet(np.ones(len(vocab)))
    lines += [f"{np.log10(p):.6f}\t{w}" for w, p in zip(vocab, lp)] + ["", "\\end\\", ""]
    t = build_ctc_topo_compact(inv) if kw.get("compact", True) else build_ctc_topo_normal(inv)
    l = build_lexicon_fst(entries, inv, words)
    g = build_grammar_fst(parse_arpa("\n".join(lines)), words)
    return t, l, g, build_tlg(t, l, g)


@pytest.mark.parametrize("seed", range(8))
def test_native_compose_matches_reference_build_tlg(seed):
    from paper_2311_04996_b200 import synth

    t, l, g, want = _ref_toy(seed, num_units=2 + seed % 4, num_words=3 + seed % 6, compact=seed % 2 == 0)
    F = synth.Fst.from_wfst
    got = synth.build_tlg(F(t), F(l), F(g)).to_wfst()
    assert _same(got, want)


@pytest.mark.parametrize("order", [1, 2, 3, 4])
def test_grammar_fst_matches_reference_parser(order):
    from ctcwfst.arpa import build_grammar_fst, parse_arpa
    from ctcwfst.wfst import SymbolTable

    from paper_2311_04996_b200 import synth

    s = synth.build_system(synth.SystemSpec(num_units=12, num_words=40, order=order, seed=3))
    words = SymbolTable()
    for i in range(1, 41):
        words.add(f"w{i}")
    ref = build_grammar_fst(parse_arpa(s.model.to_arpa(lambda i: f"w{i}")), words)
    assert _same(s.g.to_wfst(), ref)


def test_synth_tlg_flattens_like_reference():
    """FlatGraph arrays of a synthetic TLG equal the reference's flatten()."""
    from ctcwfst.decoder import flatten as ref_flatten

    from paper_2311_04996_b200 import synth

    s = synth.build_system(synth.SystemSpec(num_units=10, num_words=25, order=2, seed=4))
    rf = ref_flatten(_to_ref(s.tlg))
    fg = s.graph
    for k in ("off", "eps_end", "ilabel", "olabel", "weight", "nextstate", "final"):
        assert np.array_equal(getattr(fg, k), getattr(rf, k)), k
    assert (fg.start, fg.max_ilabel, fg.max_olabel) == (rf.start, rf.max_ilabel, rf.max_olabel)


def _to_ref(f):
    from ctcwfst.wfst import Arc, Wfst

    g = Wfst(num_states=f.num_states, start=f.start)
    for s in range(f.num_states):
        for k in range(f.off[s], f.off[s + 1]):
            g.add_arc(s, Arc(int(f.ilabel[k]), int(f.olabel[k]), float(f.weight[k]), int(f.nextstate[k])))
        if np.isfinite(f.final[s]):
            g.set_final(s, float(f.final[s]))
    return g
