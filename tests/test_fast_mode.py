"""GPU parity of the fast search mode (``search="fast"``, ctw_kernels.cu
"fast search mode"): the north star's bar -- best-path words bit-exact,
best-path cost within 1e-4 relative -- against the CPU oracle
(oracle/ctw_oracle.c, pinned to the reference in test_oracle.py) and against
the exact mode (itself identical to the reference record for record,
test_gpu_parity.py). Also: the fast kernel really ran (launch counters), it
is deterministic and chunk-invariant (streaming == offline bit for bit), and
lanes it cannot serve fall back to the exact mode.
"""

import math
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import GoldenGraph, golden_chunks, golden_names, load_golden

pytestmark = pytest.mark.gpu

COST_RTOL = 1e-4  # north_star: best-path cost within 1e-4 relative


def _system(**kw):
    from paper_2311_04996_b200 import synth

    return synth.build_system(synth.SystemSpec(**kw))


def _fast_launches(graph, cfg):
    from paper_2311_04996_b200 import flatten

    fg = flatten(graph)
    return fg.device_graph(None).pool(cfg, fg.num_states, "fast").search_info()["fast_launches"]


def _same(h, words, cost):
    assert h.words == words
    assert math.isclose(h.total_cost, cost, rel_tol=COST_RTOL, abs_tol=1e-9)


@pytest.mark.parametrize("seed", range(12))
def test_random_systems_words_match_oracle(oracle_mod, seed):
    from paper_2311_04996_b200 import DecoderConfig, DecodeState, best_path, synth

    spec = dict(num_units=4 + 3 * seed, num_words=10 + 7 * seed, order=1 + seed % 3, seed=seed,
                min_pron=1, max_pron=5)
    s = _system(**spec)
    rng = np.random.default_rng(seed)
    if seed % 2:
        frames = rng.normal(-3.0, 2.5, size=(60, spec["num_units"]))
    else:
        frames = synth.planted_utterances(s, 1, 60, seed=seed)[0]
    cfg = DecoderConfig(beam=[4.0, 9.0, 17.0, 1e9][seed % 4], max_active=[7, 60, 10_000, 300][seed % 4])
    before = _fast_launches(s.graph, cfg)
    ch = DecodeState(s.graph, cfg, search="fast")
    step = [60, 1, 7, 13][seed % 4]
    for i in range(0, 60, step):
        ch.advance_frames(frames[i:i + step])
    assert _fast_launches(s.graph, cfg) > before  # the fast kernel served these chunks
    ow, oc, ofc = oracle_mod.decode_utterance(s.graph, cfg, frames)
    h = best_path(ch)
    _same(h, ow, oc)
    assert h.frame_count == ofc
    # survivors per frame: the same count as the reference (same beam / max_active outcome)
    oh = oracle_mod.OracleChannel.from_config(s.graph, cfg)
    oh.advance_frames(frames)
    assert [len(f) for f in ch.history_records()] == [len(f) for f in oh.history_records()]


@pytest.mark.parametrize("name", [n for n in golden_names() if not n.startswith("kat_eps_cycle")])
def test_golden_words_and_costs(name):
    """Every golden fixture the fast mode can serve: same words, same cost,
    same error frame."""
    from paper_2311_04996_b200 import DecodeError, DecoderConfig, DecodeState, best_path, flatten

    d = load_golden(name)
    cfg = DecoderConfig(beam=d["beam"], max_active=d["max_active"], acoustic_scale=d["acoustic_scale"],
                        nonemitting_relax_epsilon=d["relax_eps"],
                        max_nonemitting_iters=None if d["max_ne_iters"] < 0 else d["max_ne_iters"])
    ch = DecodeState(flatten(GoldenGraph(d)), cfg, search="fast")
    if d["has_boost"]:
        ch.set_boost(d["boost"])
    err = ""
    for c in golden_chunks(d):
        try:
            ch.advance_frames(c)
        except DecodeError as e:
            err = str(e)
            break
    assert err == d["error"]
    if d["frame_count"]:
        h = best_path(ch)
        assert list(h.words) == d["best_words"].tolist()
        assert math.isclose(h.total_cost, d["best_cost"], rel_tol=COST_RTOL, abs_tol=1e-9)
        assert h.frame_count == d["frame_count"]


def test_trigram_batch_with_boosts_matches_oracle(oracle_mod):
    """Mid-size 3-gram TLG, 24 utterances in one launch, max_active binding,
    every other utterance boosted."""
    from paper_2311_04996_b200 import BoostTable, DecoderConfig, boost_costs, decode_batch, synth

    s = _system(num_units=129, blank_id=128, num_words=400, order=3, seed=5, min_pron=1, max_pron=4,
                followers=20)
    utts = list(synth.conformer_logprobs(s, 24, 120, seed=3, delta=5.0, sigma=1.5, dtype=np.float32))
    rng = np.random.default_rng(2)
    boosts = []
    for i in range(24):
        ids = rng.choice(np.arange(1, 401), size=40, replace=False)
        tab = BoostTable(entries={int(w): -float(rng.uniform(0.5, 7.0)) for w in ids})
        boosts.append(boost_costs(tab, s.graph.max_olabel) if i % 2 else None)
    cfg = DecoderConfig(beam=14.0, max_active=700)
    got = decode_batch(s.graph, cfg, utts, boost=boosts, search="fast")
    exact = decode_batch(s.graph, cfg, utts, boost=boosts)
    for u, b, h, e in zip(utts, boosts, got, exact):
        ow, oc, _ = oracle_mod.decode_utterance(s.graph, cfg, u.astype(np.float64), boost=b)
        _same(h, ow, oc)
        _same(e, ow, oc)


def test_streaming_equals_offline_bit_exact():
    from paper_2311_04996_b200 import BatcherConfig, Chunk, DecoderConfig, StreamPool, decode_batch, synth

    s = _system(num_units=30, num_words=50, order=2, seed=2)
    utts = synth.planted_utterances(s, 5, 70, seed=8)
    cfg = DecoderConfig(beam=14.0, max_active=500)
    offline = decode_batch(s.graph, cfg, utts, search="fast")
    for chunk in (1, 7, 60):
        pool = StreamPool(s.graph, cfg, BatcherConfig(max_batch=3), search="fast")
        sids = [pool.create_stream() for _ in utts]
        for sid, u in zip(sids, utts):
            for i in range(0, len(u), chunk):
                pool.push_chunk(Chunk(sid, u[i:i + chunk], is_last=i + chunk >= len(u)))
        finals = pool.drain()
        for sid, want in zip(sids, offline):
            assert finals[sid] == want


def test_deterministic_across_runs_and_lane_order():
    from paper_2311_04996_b200 import DecoderConfig, decode_batch, synth

    s = _system(num_units=129, blank_id=128, num_words=300, order=3, seed=11, min_pron=1, max_pron=4,
                followers=15)
    utts = list(synth.conformer_logprobs(s, 16, 80, seed=9, delta=5.0, sigma=1.5, dtype=np.float32))
    cfg = DecoderConfig(beam=15.0, max_active=400)
    a = decode_batch(s.graph, cfg, utts, search="fast")
    b = decode_batch(s.graph, cfg, utts[::-1], search="fast")[::-1]
    c = decode_batch(s.graph, cfg, utts, search="fast", max_lanes=5)
    assert a == b == c


def test_edge_cases_match_oracle(oracle_mod):
    """Ragged lengths, frames wider than the shared-memory row, NaN
    log-likelihoods, extreme beam / max_active, a dead frame."""
    from paper_2311_04996_b200 import DecodeFailure, DecoderConfig, decode_batch, synth

    s = _system(num_units=12, num_words=30, order=2, seed=6, min_pron=1, max_pron=4)
    rng = np.random.default_rng(1)
    base = synth.planted_utterances(s, 6, 50, seed=4, gap=4.0, noise=1.0)
    ragged = [u[: int(rng.integers(1, 50))] for u in base]
    wide = [np.concatenate([u, rng.normal(-9.0, 1.0, size=(len(u), 5000 - u.shape[1]))], axis=1) for u in base[:3]]
    nanu = base[3].copy()
    nanu[5, :4] = np.nan
    dead = base[4].copy()
    dead[7] = -np.inf
    cases = [(ragged, DecoderConfig(beam=12.0, max_active=200)),
             (wide, DecoderConfig(beam=12.0, max_active=200)),
             ([nanu, dead], DecoderConfig(beam=12.0, max_active=200)),
             (base[:3], DecoderConfig(beam=1e-6, max_active=1)),
             (base[:3], DecoderConfig(beam=1e9, max_active=1_000_000))]
    for utts, cfg in cases:
        got = decode_batch(s.graph, cfg, utts, search="fast")
        for u, h in zip(utts, got):
            try:
                want = oracle_mod.decode_utterance(s.graph, cfg, np.asarray(u, np.float64))
            except oracle_mod.OracleError:
                assert isinstance(h, DecodeFailure)
                continue
            _same(h, want[0], want[1])
            assert h.frame_count == want[2]


def test_negative_epsilon_weights_fall_back_to_exact(oracle_mod):
    """A graph with a negative epsilon weight breaks the fast mode's early
    pruning: every launch must run the exact kernel (and stay correct)."""
    from paper_2311_04996_b200 import DecodeFailure, DecoderConfig, FlatGraph, decode_batch, synth

    s = _system(num_units=10, num_words=15, order=2, seed=3)
    fg = s.graph
    w = fg.weight.copy()
    eps = np.zeros(fg.num_arcs, bool)
    for st in range(fg.num_states):
        eps[fg.off[st]:fg.eps_end[st]] = True
    k = np.flatnonzero(eps)[0]
    w[k] = -0.25
    from types import SimpleNamespace

    neg = FlatGraph.from_csr(SimpleNamespace(num_states=fg.num_states, start=fg.start, off=fg.off,
                                             eps_end=fg.eps_end, ilabel=fg.ilabel, olabel=fg.olabel, weight=w,
                                             nextstate=fg.nextstate, final=fg.final, max_ilabel=fg.max_ilabel,
                                             max_olabel=fg.max_olabel))
    utts = synth.planted_utterances(s, 3, 30, seed=1)
    cfg = DecoderConfig(beam=10.0, max_active=300)
    got = decode_batch(neg, cfg, utts, search="fast")
    assert _fast_launches(neg, cfg) == 0
    for u, h in zip(utts, got):
        try:
            ow, oc, _ = oracle_mod.decode_utterance(neg, cfg, u)
        except oracle_mod.OracleError:
            assert isinstance(h, DecodeFailure)
            continue
        assert h.words == ow and h.total_cost == oc


def test_phrase_boost_fast_equals_exact():
    from paper_2311_04996_b200 import DecoderConfig, PhraseBoost, decode_batch, synth

    s = _system(num_units=20, num_words=40, order=2, seed=12, min_pron=1, max_pron=3)
    utts = synth.planted_utterances(s, 6, 60, seed=3, gap=4.0, noise=1.0)
    cfg = DecoderConfig(beam=12.0, max_active=300)
    plain = decode_batch(s.graph, cfg, utts)
    words = sorted({w for h in plain for w in h.words})
    rng = np.random.default_rng(0)
    phr = {(int(rng.choice(words)), int(rng.choice(words))): float(rng.uniform(1.0, 4.0)) for _ in range(8)}
    pb = PhraseBoost(phr)
    fast = decode_batch(s.graph, cfg, utts, boost=[pb] * len(utts), search="fast")
    exact = decode_batch(s.graph, cfg, utts, boost=[pb] * len(utts))
    for f, e in zip(fast, exact):
        _same(f, e.words, e.total_cost)


def test_bench_scale_fast_equals_exact():
    """The benchmark's own C2 graph (3-gram TLG, 4.5 M arcs) at beam 17 /
    max_active 10k: 16 Conformer-shaped utterances x 250 frames, fast vs the
    exact mode (== the reference record for record)."""
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench

    from paper_2311_04996_b200 import DecoderConfig, decode_batch

    s = bench.system(False, "c2")
    utts = bench.workload(s, 16, 250, 0)
    cfg = DecoderConfig(beam=bench.BEAM, max_active=bench.MAX_ACTIVE)
    fast = decode_batch(s.graph, cfg, utts, search="fast")
    exact = decode_batch(s.graph, cfg, utts)
    for f, e in zip(fast, exact):
        _same(f, e.words, e.total_cost)


@pytest.mark.parametrize("search", ["exact", "fast"])
def test_wide_and_narrow_launch_shapes_agree(monkeypatch, search):
    """Small launches run the frame kernel with 1024-thread CTAs (16 per lane;
    the 64-register build while its clusters all fit, else the 32-register
    one), full batches with 512-thread CTAs (8 per lane): same hypotheses
    and, in the exact mode, the same histories."""
    from paper_2311_04996_b200 import DecoderConfig, DecodeState, decode_batch, synth

    s = _system(num_units=129, blank_id=128, num_words=300, order=3, seed=13, min_pron=1, max_pron=4,
                followers=15)
    utts = list(synth.conformer_logprobs(s, 6, 60, seed=4, delta=5.0, sigma=1.5, dtype=np.float32))
    cfg = DecoderConfig(beam=15.0, max_active=400)
    wide = decode_batch(s.graph, cfg, utts, search=search)  # 6 lanes: the 64-register wide build
    monkeypatch.setenv("CTW_NO_WIDE64", "1")
    wide32 = decode_batch(s.graph, cfg, utts, search=search)
    monkeypatch.delenv("CTW_NO_WIDE64")
    monkeypatch.setenv("CTW_NO_WIDE", "1")
    narrow = decode_batch(s.graph, cfg, utts, search=search)
    assert wide == wide32 == narrow
    if search == "exact":
        monkeypatch.delenv("CTW_NO_WIDE")
        a = DecodeState(s.graph, cfg)
        a.advance_frames(utts[0])
        monkeypatch.setenv("CTW_NO_WIDE", "1")
        b = DecodeState(s.graph, cfg)
        b.advance_frames(utts[0])
        from conftest import history_signature

        assert history_signature(a.history_records()) == history_signature(b.history_records())
