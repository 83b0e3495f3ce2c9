"""Phrase (multi-word) boosting: the Aho-Corasick automaton against brute
force on the CPU; lattice rescoring with it against path enumeration on the
GPU. One-word phrases are the reference's word boost (boosting.py:58-67:
every arc with that output label pays the table cost); longer phrases are
beyond the reference."""

import random
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))


def test_automaton_matches_brute_force():
    import lattice_oracle as lo

    from paper_2311_04996_b200 import PhraseBoost

    rng = random.Random(0)
    for _ in range(400):
        phr = {}
        for _ in range(rng.randint(1, 6)):
            ph = tuple(rng.randint(1, 4) for _ in range(rng.randint(1, 3)))
            phr[ph] = phr.get(ph, 0.0) + rng.uniform(0.5, 3.0)
        pb = PhraseBoost(phr)
        w = [rng.randint(1, 5) for _ in range(rng.randint(0, 12))]
        assert abs(pb.cost(w) - lo.phrase_cost(w, phr)) <= 1e-9


def test_bad_phrases():
    from paper_2311_04996_b200 import PhraseBoost

    with pytest.raises(ValueError):
        PhraseBoost({(): 1.0})
    with pytest.raises(ValueError):
        PhraseBoost({(0, 3): 1.0})


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(3))
def test_lattice_rescoring_matches_enumeration(seed):
    import lattice_oracle as lo

    from paper_2311_04996_b200 import DecoderConfig, PhraseBoost, decode_lattices, synth

    s = synth.build_system(synth.SystemSpec(num_units=10, num_words=30, order=2, seed=7 + seed, min_pron=1,
                                            max_pron=3))
    frames = synth.planted_utterances(s, 1, 10, seed=30 + seed, gap=3.0, noise=1.0)[0]
    cfg = DecoderConfig(beam=12.0, max_active=200)
    beam = 3.0
    lat = decode_lattices(s.graph, cfg, [frames], lattice_beam=beam)[0]
    plain = lat.nbest(20)
    rng = np.random.default_rng(seed)
    # phrases built from the lattice's own alternatives so they matter
    words = sorted({w for h in plain for w in h.words})
    phr = {}
    for h in plain[1:6]:
        if len(h.words) >= 2:
            i = int(rng.integers(0, len(h.words) - 1))
            phr[tuple(h.words[i:i + 2])] = float(rng.uniform(1.0, 4.0))
    for w in words[:3]:
        phr[(w,)] = float(rng.uniform(0.5, 2.0))
    pb = PhraseBoost(phr)
    got = lat.nbest(8, phrases=pb)
    # oracle: every complete path of the kept lattice, plus brute-force phrase costs
    import oracle as orc

    ch = orc.OracleChannel.from_config(s.graph, cfg)
    seeds = [(int(st), float(c), tuple(int(x) for x in ch.act_chain_pool[ch.act_chain_off[k]:ch.act_chain_off[k + 1]]))
             for k, (st, c) in enumerate(zip(ch.act_state, ch.act_cost))]
    ch.advance_frames(frames)
    recs = [[(r[2], r[3]) for r in fr] for fr in ch.history_records()]
    ora = lo.lattice(s.graph, cfg.acoustic_scale, np.asarray(frames, np.float64), seeds, recs, beam)
    want = lo.nbest(ora, lo.kept(ora, beam), seeds, 8, np.asarray(s.graph.final, np.float64),
                    bound=float("inf"), phrases=phr)
    assert got and want
    for (w, c), h in zip(want, got):
        assert abs(c - h.total_cost) <= 1e-3  # north_star n-best tolerance
    wmap = dict(want)
    for h in got:
        if h.words in wmap:
            assert abs(wmap[h.words] - h.total_cost) <= 1e-3
    # consistency with the plain n-best: rescoring = plain cost + phrase cost
    pmap = {h.words: h.total_cost for h in lat.nbest(200)}
    for h in got:
        if h.words in pmap:
            assert abs(pmap[h.words] + pb.cost(h.words) - h.total_cost) <= 1e-9


def _compose_oracle(s, pb):
    from paper_2311_04996_b200 import synth

    b = pb.to_fst(s.graph.max_olabel)
    tlgb = synth.arc_sort(synth.connect(synth.compose(s.tlg, b)))
    return tlgb.to_flat()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(4))
def test_in_search_phrase_boost_matches_explicit_composition(seed):
    """Phrase automaton composed inside the search == decoding the explicit
    composition TLG o B (reference compose semantics, wfst.py:307-366):
    identical words, cost within 1e-9 relative (B's weight is added after the
    arc weight instead of folded into it)."""
    from paper_2311_04996_b200 import DecoderConfig, PhraseBoost, decode_batch, synth

    s = synth.build_system(synth.SystemSpec(num_units=10, num_words=25, order=2, seed=11 + seed, min_pron=1,
                                            max_pron=3))
    utts = synth.planted_utterances(s, 6, 40, seed=40 + seed, gap=4.0, noise=1.0)
    cfg = DecoderConfig(beam=14.0, max_active=10_000)
    rng = np.random.default_rng(seed)
    plain = decode_batch(s.graph, cfg, utts)
    phr = {}
    for h in plain[:4]:
        if len(h.words) >= 2:
            i = int(rng.integers(0, len(h.words) - 1))
            phr[tuple(h.words[i:i + 2])] = float(rng.uniform(1.0, 5.0))
    phr[(int(rng.integers(1, 26)), int(rng.integers(1, 26)))] = 3.0
    phr[(int(rng.integers(1, 26)),)] = 1.5
    pb = PhraseBoost(phr)
    assert not pb.single_words
    got = decode_batch(s.graph, cfg, utts, boost=[pb] * len(utts))
    want = decode_batch(_compose_oracle(s, pb), cfg, utts)
    for g, w in zip(got, want):
        assert g.words == w.words
        assert abs(g.total_cost - w.total_cost) <= 1e-9 * max(1.0, abs(w.total_cost))


@pytest.mark.gpu
def test_single_word_phrases_are_the_word_boost():
    from paper_2311_04996_b200 import DecoderConfig, PhraseBoost, decode_batch, synth

    s = synth.build_system(synth.SystemSpec(num_units=10, num_words=25, order=2, seed=3, min_pron=1, max_pron=3))
    utts = synth.planted_utterances(s, 4, 40, seed=9, gap=4.0, noise=1.0)
    cfg = DecoderConfig(beam=14.0, max_active=300)
    pb = PhraseBoost({(3,): 2.0, (7,): 1.0, (11,): 4.0})
    assert pb.single_words
    dense = pb.word_costs(s.graph.max_olabel + 1)
    assert decode_batch(s.graph, cfg, utts, boost=[pb] * 4) == decode_batch(s.graph, cfg, utts, boost=dense)


@pytest.mark.gpu
def test_lattice_of_phrase_boosted_decode():
    """Lattices of lanes decoded with an in-search phrase automaton: the
    lattice's best path is the boosted decode's best path and its 1-best
    equals it."""
    from paper_2311_04996_b200 import DecoderConfig, PhraseBoost, decode_batch, decode_lattices, synth

    s = synth.build_system(synth.SystemSpec(num_units=10, num_words=25, order=2, seed=12, min_pron=1, max_pron=3))
    utts = synth.planted_utterances(s, 4, 30, seed=8, gap=4.0, noise=1.0)
    cfg = DecoderConfig(beam=14.0, max_active=500)
    plain = decode_batch(s.graph, cfg, utts)
    phr = {tuple(h.words[:2]): 2.5 for h in plain if len(h.words) >= 2}
    pb = PhraseBoost(phr)
    hyps = decode_batch(s.graph, cfg, utts, boost=[pb] * 4)
    lats = decode_lattices(s.graph, cfg, utts, lattice_beam=4.0, boost=[pb] * 4)
    for lat, h in zip(lats, hyps):
        assert lat.status == 0
        assert lat.best_path == h
        assert abs(lat.best_cost - h.total_cost) <= 1e-9
        assert lat.nbest(2)[0].words == h.words


def test_fsa_too_large_for_graph_is_rejected():
    from paper_2311_04996_b200 import PhraseBoost

    pb = PhraseBoost({tuple(range(1, 40)): 1.0})
    assert pb.num_states == 40


@pytest.mark.gpu
def test_streaming_with_phrase_boost_equals_offline():
    from paper_2311_04996_b200 import (BatcherConfig, Chunk, DecoderConfig, PhraseBoost, StreamPool, decode_batch,
                                       synth)

    s = synth.build_system(synth.SystemSpec(num_units=10, num_words=25, order=2, seed=12, min_pron=1, max_pron=3))
    utts = synth.planted_utterances(s, 4, 45, seed=5, gap=4.0, noise=1.0)
    cfg = DecoderConfig(beam=14.0, max_active=500)
    plain = decode_batch(s.graph, cfg, utts)
    pb = PhraseBoost({tuple(h.words[:2]): 2.0 for h in plain if len(h.words) >= 2})
    offline = decode_batch(s.graph, cfg, utts, boost=[pb] * len(utts))
    pool = StreamPool(s.graph, cfg, BatcherConfig(max_batch=2))
    sids = [pool.create_stream(pb) for _ in utts]
    for sid, u in zip(sids, utts):
        for i in range(0, len(u), 7):
            pool.push_chunk(Chunk(sid, u[i:i + 7], is_last=i + 7 >= len(u)))
    finals = pool.drain()
    for sid, want in zip(sids, offline):
        assert finals[sid] == want
