"""Lattice generation / pruning / n-best on the GPU against the CPU
restatement of the lattice definition (oracle/lattice_oracle.py) and a
brute-force path enumeration. The lattice's nodes are the decoder's records
(pinned to the reference), its best complete path must be best_path's, and
n-best scores must match the enumeration within 1e-3 absolute (BASELINE.json
north_star)."""

import math
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))

NBEST_TOL = 1e-3  # north_star: lattice / n-best scores within 1e-3 absolute
W_TOL = 1e-9      # arc weights: same operation order, only closure paths may differ in rounding


def _system(**kw):
    from paper_2311_04996_b200 import synth

    return synth.build_system(synth.SystemSpec(**kw))


def _oracle_lattice(s, cfg, frames, beam, boost=None):
    import lattice_oracle as lo
    import oracle as orc

    ch = orc.OracleChannel.from_config(s.graph, cfg, boost=boost)
    seeds = [(int(st), float(c), tuple(int(x) for x in ch.act_chain_pool[ch.act_chain_off[k]:ch.act_chain_off[k + 1]]))
             for k, (st, c) in enumerate(zip(ch.act_state, ch.act_cost))]
    ch.advance_frames(frames)
    recs = [[(r[2], r[3]) for r in fr] for fr in ch.history_records()]
    lat = lo.lattice(s.graph, cfg.acoustic_scale, np.asarray(frames, np.float64), seeds, recs, beam, boost)
    return lat, seeds, ch.best_path()


def _key(layer, state):
    return (layer, state)


def _gpu_arcs(lat):
    seed_state = {k: int(s) for k, s in enumerate(lat.seed_state)}
    out = []
    for k in range(lat.num_arcs):
        f = int(lat.frame[k])
        src = (f - 1, int(lat.src_state[k]))
        if int(lat.src[k]) < len(seed_state):
            assert f == 0 and seed_state[int(lat.src[k])] == int(lat.src_state[k])
        out.append((f, src, (f, int(lat.dst_state[k])), float(lat.weight[k]), lat.labels[k]))
    return out


def _oracle_arcs(arcs, alpha_state):
    return [(f, alpha_state[src], (f, y), w, labs) for f, src, d, y, w, labs, score in arcs]


def _match(gpu, ora):
    """Multisets of (frame, src key, dst key, labels) with weights within W_TOL."""
    from collections import defaultdict

    g, o = defaultdict(list), defaultdict(list)
    for f, s, d, w, l in gpu:
        g[(f, s, d, l)].append(w)
    for f, s, d, w, l in ora:
        o[(f, s, d, l)].append(w)
    return g, o


SPECS = [
    dict(num_units=8, num_words=20, order=2, seed=1),
    dict(num_units=12, num_words=40, order=3, seed=4, min_pron=1, max_pron=4),
    dict(num_units=10, num_words=30, order=2, seed=7, min_pron=1, max_pron=3),
]


@pytest.mark.parametrize("search", ["exact", "fast"])
@pytest.mark.parametrize("k", range(len(SPECS)))
@pytest.mark.parametrize("beam", [0.0, 3.0, 8.0])
def test_lattice_matches_oracle(k, beam, search):
    """(The fast mode keeps the same survivors with the same costs, so its
    lattice is the same lattice.)"""
    import lattice_oracle as lo

    from paper_2311_04996_b200 import DecoderConfig, decode_lattices, synth

    s = _system(**SPECS[k])
    frames = synth.planted_utterances(s, 1, 30, seed=10 + k, gap=3.0, noise=1.0)[0]
    cfg = DecoderConfig(beam=14.0, max_active=400)
    lat = decode_lattices(s.graph, cfg, [frames], lattice_beam=beam, search=search)[0]
    ora, seeds, (ow, oc, _) = _oracle_lattice(s, cfg, frames, beam)
    assert lat.status == 0
    # the lattice's best complete path is the decoder's best path
    assert math.isclose(lat.best_cost, lat.best_path.total_cost, rel_tol=0, abs_tol=1e-9)
    assert lat.best_path.words == ow and abs(oc - lat.best_cost) <= 1e-9
    assert abs(ora["best"] - lat.best_cost) <= 1e-9
    # node identity: (layer, state); oracle node id -> key
    node_key = {}
    for i, (st, _, _) in enumerate(seeds):
        node_key[i] = (-1, st)
    for f, src, d, y, w, labs, score in ora["arcs"]:
        node_key[d] = (f, y)
    # GPU arcs must contain every oracle arc inside the beam (minus rounding
    # slack) and only oracle arcs inside the beam (plus slack)
    inner = lo.kept(ora, beam, -1e-7)
    outer = lo.kept(ora, beam, +1e-7)
    gpu = _gpu_arcs(lat)
    gset = {}
    for f, s_, d, w, l in gpu:
        gset.setdefault((f, s_, d, l), []).append(w)
    oset_outer = {}
    for f, src, d, y, w, labs, score in outer:
        oset_outer.setdefault((f, node_key.get(src, (f - 1, None)), (f, y), labs), []).append(w)
    for f, src, d, y, w, labs, score in inner:
        key = (f, node_key.get(src, (f - 1, None)), (f, y), labs)
        assert key in gset, ("missing arc", key, w, score)
        assert min(abs(w - x) for x in gset[key]) <= W_TOL
    for key, ws in gset.items():
        assert key in oset_outer, ("extra arc", key, ws)
    assert len(gpu) >= len(inner)
    assert len(gpu) <= len(outer)


@pytest.mark.parametrize("k", range(len(SPECS)))
def test_nbest_matches_enumeration(k):
    import lattice_oracle as lo

    from paper_2311_04996_b200 import DecoderConfig, decode_lattices, synth

    s = _system(**SPECS[k])
    frames = synth.planted_utterances(s, 1, 10, seed=20 + k, gap=3.0, noise=1.0)[0]
    cfg = DecoderConfig(beam=12.0, max_active=200)
    beam = 3.0
    lat = decode_lattices(s.graph, cfg, [frames], lattice_beam=beam)[0]
    got = lat.nbest(8)
    ora, seeds, _ = _oracle_lattice(s, cfg, frames, beam)
    want = lo.nbest(ora, lo.kept(ora, beam), seeds, 8, np.asarray(s.graph.final, np.float64),
                    bound=ora["best"] + beam)
    got = [h for h in got if h.total_cost <= ora["best"] + beam - 1e-6]
    assert got and want
    # best first, the decoder's best path on top
    assert got[0].words == lat.best_path.words
    assert abs(got[0].total_cost - lat.best_path.total_cost) <= 1e-9
    assert all(a.total_cost <= b.total_cost + 1e-12 for a, b in zip(got, got[1:]))
    # same word sequences with scores within the north-star tolerance
    # (sequences whose scores tie within the tolerance may swap places)
    wmap = dict(want)
    for h in got:
        if h.words in wmap:
            assert abs(wmap[h.words] - h.total_cost) <= NBEST_TOL
    common = [h for h in got if h.words in wmap]
    assert len(common) >= min(len(got), len(want)) - 1
    for (w1, c1), h in zip(want, got):
        assert abs(c1 - h.total_cost) <= NBEST_TOL


def test_lattice_batch_and_boost():
    """A batch of utterances in one launch (some boosted): every lattice's best
    path equals decode_batch's, 1-best of n-best equals the best path."""
    from paper_2311_04996_b200 import DecoderConfig, decode_batch, decode_lattices, synth

    s = _system(num_units=12, num_words=40, order=3, seed=4, min_pron=1, max_pron=4)
    utts = synth.planted_utterances(s, 6, 40, seed=3, gap=3.0, noise=1.0)
    cfg = DecoderConfig(beam=14.0, max_active=300)
    rng = np.random.default_rng(0)
    boosts = []
    for i in range(6):
        if i % 2:
            b = np.zeros(s.graph.max_olabel + 1)
            b[rng.choice(np.arange(1, 41), 5, replace=False)] = -rng.uniform(0.5, 3.0, 5)
            boosts.append(b)
        else:
            boosts.append(None)
    lats = decode_lattices(s.graph, cfg, utts, lattice_beam=5.0, boost=boosts)
    hyps = decode_batch(s.graph, cfg, utts, boost=boosts)
    for lat, h in zip(lats, hyps):
        assert lat.best_path == h
        assert abs(lat.best_cost - h.total_cost) <= 1e-9
        nb = lat.nbest(3)
        assert nb[0].words == h.words
        assert lat.num_arcs > 0


def test_nbest_lattices_pool_matches_serial():
    """nbest_lattices (host thread pool) returns each lattice's own n-best."""
    from paper_2311_04996_b200 import DecoderConfig, decode_lattices, nbest_lattices, synth

    s = _system(num_units=12, num_words=40, order=3, seed=4, min_pron=1, max_pron=4)
    utts = synth.planted_utterances(s, 8, 30, seed=9, gap=3.0, noise=1.0)
    lats = decode_lattices(s.graph, DecoderConfig(beam=14.0, max_active=300), utts, lattice_beam=4.0)
    serial = [lat.nbest(5) for lat in lats]
    pooled = nbest_lattices(lats, 5, workers=4)
    assert [[(h.words, h.total_cost) for h in x] for x in pooled] == \
        [[(h.words, h.total_cost) for h in x] for x in serial]


def test_wide_epsilon_closure_reruns_with_large_capacity():
    """A hub state with 60 epsilon arcs: a work item's local closure outgrows
    the fast kernel's 48 entries (status 3), the host re-runs the lane with
    the large-capacity kernel, and the lattice equals the CPU restatement's
    (never a silently truncated lattice)."""
    import lattice_oracle as lo

    from paper_2311_04996_b200 import DecoderConfig, FlatGraph, decode_lattices

    n_leaf = 60
    src, il, ol, w, ns = [0], [1], [1], [0.5], [1]
    for k in range(2, 2 + n_leaf):
        src += [1, k]
        il += [0, 1 + k % 3]
        ol += [k, 0]
        w += [0.01 * k, 0.1]
        ns += [k, 1]
    final = np.full(2 + n_leaf, np.inf)
    final[2:] = 0.0
    fg = FlatGraph.from_arrays(2 + n_leaf, 0, src, il, ol, w, ns, final)

    class Sys:
        graph = fg

    rng = np.random.default_rng(3)
    frames = rng.normal(-1.0, 0.5, size=(6, 4))
    cfg = DecoderConfig(beam=1e9, max_active=10_000)
    beam = 1.5
    lat = decode_lattices(fg, cfg, [frames], lattice_beam=beam)[0]
    assert lat.status == 0
    ora, seeds, (ow, oc, _) = _oracle_lattice(Sys, cfg, frames, beam)
    assert lat.best_path.words == ow and abs(lat.best_cost - oc) <= 1e-9
    inner = lo.kept(ora, beam, -1e-7)
    outer = lo.kept(ora, beam, +1e-7)
    assert len(inner) <= lat.num_arcs <= len(outer)


def test_lattice_cluster_split_matches_single_cta(monkeypatch):
    """The lattice kernel spreads a lane over up to 8 CTAs (a cluster) when
    the batch leaves SMs idle: the lattices equal the one-CTA-per-lane ones
    arc for arc."""
    from paper_2311_04996_b200 import DecoderConfig, decode_lattices, synth

    s = _system(num_units=129, blank_id=128, num_words=300, order=3, seed=5, min_pron=1, max_pron=4,
                followers=15)
    utts = list(synth.conformer_logprobs(s, 12, 80, seed=2, delta=5.0, sigma=1.5, dtype=np.float32))
    cfg = DecoderConfig(beam=14.0, max_active=500)
    out = {}
    for r in ("1", "8"):
        monkeypatch.setenv("CTW_LAT_RANKS", r)
        out[r] = decode_lattices(s.graph, cfg, utts, lattice_beam=5.0)
    def canon(lat):  # node ids follow the decoder's (free) record order: compare by (layer, state)
        return sorted(zip(lat.frame.tolist(), lat.src_state.tolist(), lat.dst_state.tolist(), lat.weight.tolist(),
                          lat.labels))

    for a, b in zip(out["1"], out["8"]):
        assert a.num_arcs == b.num_arcs > 0
        assert canon(a) == canon(b)
        # same n-best up to f64 summation order (the search adds arc weights
        # in node order, and node ids follow the free record order)
        na, nb = a.nbest(5), b.nbest(5)
        assert len(na) == len(nb)
        for x, y in zip(na, nb):
            assert abs(x.total_cost - y.total_cost) <= 1e-9 * abs(x.total_cost)
        assert {h.words for h in na} == {h.words for h in nb} or \
            abs(na[-1].total_cost - na[-2].total_cost) <= 1e-9 * abs(na[-1].total_cost)


def _canon(lat):
    return sorted(zip(lat.frame.tolist(), lat.src_state.tolist(), lat.dst_state.tolist(), lat.labels,
                      lat.weight.tolist()))


@pytest.mark.parametrize("search", ["exact", "fast"])
def test_closure_index_matches_general_kernel(monkeypatch, search):
    """Graphs whose epsilon arcs carry no output label take the indexed
    lattice kernel (closures from the per-graph closure index, destinations
    from a shared-memory map). Its lattices equal the general kernel's
    (per-item closures) arc for arc; weights agree up to the summation order
    c0 + (w1 + w2) vs (c0 + w1) + w2."""
    from paper_2311_04996_b200 import DecoderConfig, decode_lattices, synth

    s = _system(num_units=129, blank_id=128, num_words=300, order=3, seed=5, min_pron=1, max_pron=4,
                followers=15)
    fg = s.graph
    eps = np.concatenate([np.arange(fg.off[i], fg.eps_end[i]) for i in range(fg.num_states)])
    assert len(eps) and not np.any(np.asarray(fg.olabel)[eps])  # the indexed kernel applies
    utts = list(synth.conformer_logprobs(s, 10, 80, seed=4, delta=5.0, sigma=1.5, dtype=np.float32))
    cfg = DecoderConfig(beam=14.0, max_active=500)
    rng = np.random.default_rng(1)
    boosts = []
    for i in range(len(utts)):
        b = None
        if i % 3 == 1:
            b = np.zeros(fg.max_olabel + 1)
            b[rng.choice(np.arange(1, fg.max_olabel + 1), 20, replace=False)] = -rng.uniform(0.5, 3.0, 20)
        boosts.append(b)
    out = {}
    for mode in ("pre", "general"):
        if mode == "general":
            monkeypatch.setenv("CTW_LAT_NOPRE", "1")
        out[mode] = decode_lattices(fg, cfg, utts, lattice_beam=5.0, boost=boosts, search=search)
    for a, b in zip(out["pre"], out["general"]):
        assert a.status == b.status == 0
        assert a.num_arcs == b.num_arcs > 0
        ca, cb = _canon(a), _canon(b)
        assert [x[:4] for x in ca] == [x[:4] for x in cb]
        assert all(abs(x[4] - y[4]) <= W_TOL * max(1.0, abs(y[4])) for x, y in zip(ca, cb))
        assert a.best_path == b.best_path and abs(a.best_cost - b.best_cost) <= 1e-9
        na, nb = a.nbest(5), b.nbest(5)
        assert [h.words for h in na] == [h.words for h in nb] or \
            abs(na[-1].total_cost - na[-2].total_cost) <= 1e-9 * abs(na[-1].total_cost)


def test_closure_index_overflow_reruns_general_kernel():
    """A hub with 80 unlabelled epsilon arcs: its closure is too large for the
    closure index (64 entries), items reaching it mark the lane (status 3),
    and the host re-runs it with the general large-capacity kernel; the
    lattice equals the CPU restatement's."""
    import lattice_oracle as lo

    from paper_2311_04996_b200 import DecoderConfig, FlatGraph, decode_lattices

    n_leaf = 80
    src, il, ol, w, ns = [0], [1], [1], [0.5], [1]
    for k in range(2, 2 + n_leaf):
        src += [1, k]
        il += [0, 1 + k % 3]
        ol += [0, k]
        w += [0.01 * k, 0.1]
        ns += [k, 1]
    final = np.full(2 + n_leaf, np.inf)
    final[2:] = 0.0
    fg = FlatGraph.from_arrays(2 + n_leaf, 0, src, il, ol, w, ns, final)

    class Sys:
        graph = fg

    rng = np.random.default_rng(5)
    frames = rng.normal(-1.0, 0.5, size=(6, 4))
    cfg = DecoderConfig(beam=1e9, max_active=10_000)
    beam = 1.5
    lat = decode_lattices(fg, cfg, [frames], lattice_beam=beam)[0]
    assert lat.status == 0
    ora, seeds, (ow, oc, _) = _oracle_lattice(Sys, cfg, frames, beam)
    assert lat.best_path.words == ow and abs(lat.best_cost - oc) <= 1e-9
    inner = lo.kept(ora, beam, -1e-7)
    outer = lo.kept(ora, beam, +1e-7)
    assert len(inner) <= lat.num_arcs <= len(outer)


def test_lattice_arrays_are_views_that_outlive_the_lattice():
    """Lattice arrays are zero-copy views of the C result arrays: they stay
    valid after the Lattice object is gone (the C arrays are freed with the
    last view), and equal a copy taken while the lattice was alive."""
    import gc

    from paper_2311_04996_b200 import DecoderConfig, decode_lattices, synth

    s = _system(num_units=12, num_words=40, order=3, seed=4, min_pron=1, max_pron=4)
    utts = synth.planted_utterances(s, 3, 30, seed=5, gap=3.0, noise=1.0)
    lats = decode_lattices(s.graph, DecoderConfig(beam=14.0, max_active=300), utts, lattice_beam=4.0)
    kept = [(lat.weight, lat.src, lat.label_pool) for lat in lats]
    copies = [(w.copy(), sr.copy(), lp.copy()) for w, sr, lp in kept]
    del lats
    gc.collect()
    junk = [np.full(1 << 16, 7.0) for _ in range(64)]  # reuse freed heap memory if any was freed early
    for (w, sr, lp), (w0, sr0, lp0) in zip(kept, copies):
        assert np.array_equal(w, w0) and np.array_equal(sr, sr0) and np.array_equal(lp, lp0)
    del junk


def test_closure_index_with_phrase_automaton_matches_general_kernel(monkeypatch):
    """In-search phrase automata put the automaton state in the token key's
    high bits; the indexed lattice kernel carries them through the closure
    (epsilon arcs have no labels, so the automaton state is constant along a
    closure). Its lattices equal the general kernel's arc for arc."""
    from paper_2311_04996_b200 import DecoderConfig, PhraseBoost, decode_batch, decode_lattices, synth

    s = synth.build_system(synth.SystemSpec(num_units=10, num_words=25, order=2, seed=12, min_pron=1, max_pron=3))
    utts = synth.planted_utterances(s, 4, 30, seed=8, gap=4.0, noise=1.0)
    cfg = DecoderConfig(beam=14.0, max_active=500)
    plain = decode_batch(s.graph, cfg, utts)
    pb = PhraseBoost({tuple(h.words[:2]): 2.5 for h in plain if len(h.words) >= 2})
    out = {}
    for mode in ("pre", "general"):
        if mode == "general":
            monkeypatch.setenv("CTW_LAT_NOPRE", "1")
        out[mode] = decode_lattices(s.graph, cfg, utts, lattice_beam=4.0, boost=[pb] * 4)
    for a, b in zip(out["pre"], out["general"]):
        assert a.status == b.status == 0 and a.num_arcs == b.num_arcs > 0
        ca, cb = _canon(a), _canon(b)
        assert [x[:4] for x in ca] == [x[:4] for x in cb]
        assert all(abs(x[4] - y[4]) <= W_TOL * max(1.0, abs(y[4])) for x, y in zip(ca, cb))
        assert a.best_path == b.best_path
