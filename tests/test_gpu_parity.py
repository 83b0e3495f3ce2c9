"""GPU parity: the sm_100a decoder against the reference's golden vectors and
the CPU oracle (oracle/ctw_oracle.c, itself pinned in test_oracle.py).

Bar (BASELINE.json north_star): best-path words bit-exact, best-path cost
within 1e-4 relative. The GPU computes in IEEE f64 with the reference's
operation order and resolves exact f64 ties in the reference's Gauss-Seidel
order, so these tests demand MORE: the whole
per-frame history (prev pointer, olabels, state, cost of every record) and
the active token set identical to the reference's.
"""

import math

import numpy as np
import pytest

from conftest import (GoldenGraph, assert_history_equivalent, expected_history, golden_chunks, golden_names,
                      load_golden)

pytestmark = pytest.mark.gpu

COST_RTOL = 1e-4  # north_star tolerance on best-path cost (we also check exact equality)


def _cfg(d):
    from paper_2311_04996_b200 import DecoderConfig

    return DecoderConfig(beam=d["beam"], max_active=d["max_active"], acoustic_scale=d["acoustic_scale"],
                         nonemitting_relax_epsilon=d["relax_eps"],
                         max_nonemitting_iters=None if d["max_ne_iters"] < 0 else d["max_ne_iters"])


def _run_golden(d, kernel=None):
    from paper_2311_04996_b200 import DecodeError, DecodeState, flatten

    fg = flatten(GoldenGraph(d))
    ch = DecodeState(fg, _cfg(d), kernel=kernel)
    boost = d["boost"] if d["has_boost"] else None
    if boost is not None:
        if d["boost_poke"]:
            ch.boost = boost
        else:
            ch.set_boost(boost)
    seed = sorted((t.state, t.cost) for t in ch.active_tokens())
    err = ""
    for c in golden_chunks(d):
        try:
            ch.advance_frames(c)
        except DecodeError as e:
            err = str(e)
            break
    return ch, seed, err


def _check_channel(d, ch, seed, err, name=""):
    from paper_2311_04996_b200 import best_path

    assert seed == sorted(zip(d["seed_state"].tolist(), d["seed_cost"].tolist()))
    assert err == d["error"]
    assert ch.history_records() == expected_history(d)  # every record, prev pointers included
    assert [t.state for t in ch.active_tokens()] == d["tok_state"].tolist()
    assert [t.cost for t in ch.active_tokens()] == d["tok_cost"].tolist()
    assert [t.backpointer for t in ch.active_tokens()] == d["tok_bp"].tolist()
    if d["frame_count"]:
        h = best_path(ch)
        assert list(h.words) == d["best_words"].tolist()
        assert h.total_cost == d["best_cost"]
        assert h.frame_count == d["frame_count"]


@pytest.mark.parametrize("name", golden_names())
def test_golden_native_lane(name):
    d = load_golden(name)
    ch, seed, err = _run_golden(d)
    _check_channel(d, ch, seed, err, name)


@pytest.mark.parametrize("name", golden_names())
def test_golden_through_reference_kernel_seam(name):
    """DecodeState(kernel=kernels.advance_chunk): the reference's plug-in
    contract served by the GPU."""
    from paper_2311_04996_b200 import kernels

    d = load_golden(name)
    ch, seed, err = _run_golden(d, kernel=kernels.advance_chunk)
    _check_channel(d, ch, seed, err, name)


def test_golden_decode_batch_one_launch():
    from paper_2311_04996_b200 import Hypothesis, decode_batch, flatten

    names = [n for n in golden_names() if n.startswith("c1_")]
    ds = [load_golden(n) for n in names]
    fg = flatten(GoldenGraph(ds[0]))
    got = decode_batch(fg, _cfg(ds[0]), [d["frames"] for d in ds])
    for d, h in zip(ds, got):
        assert isinstance(h, Hypothesis)
        assert list(h.words) == d["best_words"].tolist()
        assert h.total_cost == d["best_cost"]


def test_dead_beam_is_atomic_and_recoverable():
    from paper_2311_04996_b200 import DecodeError, DecodeState, flatten

    d = load_golden("kat_dead_beam")
    ch = DecodeState(flatten(GoldenGraph(d)), _cfg(d))
    frames = d["frames"]
    with pytest.raises(DecodeError, match="frame 1"):
        ch.advance_frames(frames)
    assert ch.frame_count == 0
    assert ch.active_states() == {0, 3}
    ch.advance_frames(frames[:1])
    assert ch.frame_count == 1


# ------------------------------------------------------------ vs oracle ----


def _system(**kw):
    from paper_2311_04996_b200 import synth

    return synth.build_system(synth.SystemSpec(**kw))


@pytest.mark.parametrize("seed", range(12))
def test_random_systems_history_identical_to_oracle(oracle_mod, seed):
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
    ch = DecodeState(s.graph, cfg)
    oc = oracle_mod.OracleChannel.from_config(s.graph, cfg)
    step = [60, 1, 7, 13][seed % 4]
    for i in range(0, 60, step):
        ch.advance_frames(frames[i:i + step])
        oc.advance_frames(frames[i:i + step])
    # exact costs/states/olabels and identical transcript behind every record;
    # prev pointers may differ only in the f64 rounding corner documented in
    # DESIGN.md ("Epsilon closure: residual corner")
    assert_history_equivalent(ch.history_records(), oc.history_records(), exact_prev=False)
    h = best_path(ch)
    assert (h.words, h.total_cost, h.frame_count) == oc.best_path()


def test_trigram_batch_matches_oracle(oracle_mod):
    """Mid-size 3-gram TLG, 24 utterances in one launch, max_active binding."""
    from paper_2311_04996_b200 import DecoderConfig, decode_batch, synth

    s = _system(num_units=129, blank_id=128, num_words=400, order=3, seed=5, min_pron=1, max_pron=4,
                followers=20)
    utts = list(synth.conformer_logprobs(s, 24, 120, seed=3, delta=5.0, sigma=1.5, dtype=np.float32))
    cfg = DecoderConfig(beam=14.0, max_active=700)
    got = decode_batch(s.graph, cfg, utts)
    for u, h in zip(utts, got):
        ow, oc, ofc = oracle_mod.decode_utterance(s.graph, cfg, u.astype(np.float64))
        assert h.words == ow
        assert h.total_cost == oc
        assert math.isclose(h.total_cost, oc, rel_tol=COST_RTOL)


def test_per_utterance_boost_matches_oracle(oracle_mod):
    from paper_2311_04996_b200 import BoostTable, DecoderConfig, boost_costs, decode_batch, synth

    s = _system(num_units=30, num_words=60, order=2, seed=9)
    utts = synth.planted_utterances(s, 6, 80, seed=4, gap=6.0, noise=1.5)
    rng = np.random.default_rng(0)
    boosts = []
    for i in range(6):
        ids = rng.choice(np.arange(1, 61), size=10, replace=False)
        tab = BoostTable(entries={int(w): -float(rng.uniform(0.5, 8.5)) for w in ids})
        boosts.append(boost_costs(tab, s.graph.max_olabel) if i % 3 else None)
    cfg = DecoderConfig(beam=12.0, max_active=500)
    got = decode_batch(s.graph, cfg, utts, boost=boosts)
    for u, b, h in zip(utts, boosts, got):
        ow, oc, _ = oracle_mod.decode_utterance(s.graph, cfg, u, boost=b)
        assert h.words == ow and h.total_cost == oc


def test_streaming_equals_offline_bit_exact():
    from paper_2311_04996_b200 import BatcherConfig, Chunk, DecoderConfig, StreamPool, decode_utterance, synth

    s = _system(num_units=30, num_words=50, order=2, seed=2)
    utts = synth.planted_utterances(s, 5, 70, seed=8)
    cfg = DecoderConfig(beam=14.0, max_active=500)
    offline = [decode_utterance(s.graph, cfg, u) for u in utts]
    for chunk in (1, 7, 60):
        pool = StreamPool(s.graph, cfg, BatcherConfig(max_batch=3))
        sids = [pool.create_stream() for _ in utts]
        for sid, u in zip(sids, utts):
            cuts = list(range(0, len(u), chunk))
            for i in cuts:
                pool.push_chunk(Chunk(sid, u[i:i + chunk], is_last=i + chunk >= len(u)))
        finals = pool.drain()
        for sid, want in zip(sids, offline):
            assert finals[sid] == want


def test_stream_partials_and_state_machine():
    from paper_2311_04996_b200 import BatcherConfig, Chunk, DecoderConfig, StreamError, StreamPool, synth

    s = _system(num_units=10, num_words=12, order=1, seed=4)
    pool = StreamPool(s.graph, DecoderConfig(beam=10.0, max_active=200), BatcherConfig(max_batch=1))
    sid = pool.create_stream()
    for _ in range(3):
        pool.push_chunk(Chunk(sid, np.zeros((2, 10))))
    pool.push_chunk(Chunk(sid, np.zeros((0, 10)), is_last=True))
    with pytest.raises(StreamError, match="draining"):
        pool.push_chunk(Chunk(sid, np.zeros((2, 10))))
    seen = 0
    while True:
        out = pool.step()
        if not out:
            break
        seen += 1
        assert out[0][0] == sid
        assert out[0][1].frame_count == min(seen * 2, 6)
    assert seen == 4
    assert pool.finish_stream(sid).frame_count == 6
    with pytest.raises(StreamError, match="finished"):
        pool.finish_stream(sid)


def test_api_errors_match_reference_messages():
    from paper_2311_04996_b200 import DecodeError, DecoderConfig, advance, best_path, create_channel, synth

    s = _system(num_units=6, num_words=8, order=1, seed=1)
    ch = create_channel(s.graph, DecoderConfig(beam=1e9, max_active=10**9))
    with pytest.raises(DecodeError, match="frames"):
        best_path(ch)
    ch.advance_frames(np.zeros((0, 6)))
    assert ch.frame_count == 0
    with pytest.raises(DecodeError, match="tokens"):
        ch.advance_frames(np.zeros((1, 3)))
    advance(ch, np.full(6, -1.0))
    with pytest.raises(DecodeError, match="tokens"):
        advance(ch, np.full(7, -1.0))
    with pytest.raises(DecodeError, match="before"):
        ch.set_boost(np.zeros(s.graph.max_olabel + 1))


def test_torch_cuda_tensors_zero_copy_path(oracle_mod):
    import torch

    from paper_2311_04996_b200 import DecoderConfig, decode_batch, synth

    s = _system(num_units=30, num_words=40, order=2, seed=6)
    utts = synth.planted_utterances(s, 4, 50, seed=1, dtype=np.float32)
    cfg = DecoderConfig(beam=12.0, max_active=400)
    host = decode_batch(s.graph, cfg, utts)
    dev = decode_batch(s.graph, cfg, [torch.from_numpy(u).cuda() for u in utts])
    assert host == dev
    for u, h in zip(utts, host):
        assert (h.words, h.total_cost) == oracle_mod.decode_utterance(s.graph, cfg, u.astype(np.float64))[:2]


def test_lane_reuse_and_decode_failure_per_index():
    from paper_2311_04996_b200 import DecodeFailure, DecoderConfig, Hypothesis, decode_batch, synth

    s = _system(num_units=12, num_words=20, order=2, seed=3)
    utts = synth.planted_utterances(s, 5, 30, seed=2)
    bad = utts[2].copy()
    bad[4] = -np.inf
    utts[2] = bad
    utts[3] = np.zeros((0, 12))
    cfg = DecoderConfig(beam=10.0, max_active=100)
    for _ in range(3):  # lanes are recycled between calls
        got = decode_batch(s.graph, cfg, utts)
        assert isinstance(got[0], Hypothesis) and isinstance(got[4], Hypothesis)
        assert isinstance(got[2], DecodeFailure) and "frame 4" in str(got[2].error)
        assert isinstance(got[3], DecodeFailure)


def test_bench_scale_history_matches_oracle(oracle_mod):
    """The benchmark's own graph (C2: 3-gram TLG, 4.5 M arcs) at the bench
    configuration (beam 17, max_active 10k): every record's cost, state and
    transcript equal the CPU oracle's for two Conformer-shaped utterances."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    from conftest import assert_history_equivalent

    from paper_2311_04996_b200 import DecoderConfig, DecodeState, best_path

    s = bench.system(False, "c2")
    utts = bench.workload(s, 2, 60, 0)
    cfg = DecoderConfig(beam=bench.BEAM, max_active=bench.MAX_ACTIVE)
    for u in utts:
        ch = DecodeState(s.graph, cfg)
        ch.advance_frames(u)
        oc = oracle_mod.OracleChannel.from_config(s.graph, cfg)
        oc.advance_frames(u.astype(np.float64))
        assert_history_equivalent(ch.history_records(), oc.history_records(), exact_prev=False)
        h = best_path(ch)
        assert (h.words, h.total_cost, h.frame_count) == oc.best_path()


@pytest.mark.parametrize("search", ["exact", "fast"])
def test_history_compaction_keeps_best_paths(search):
    """Partial-history garbage collection (ctw_lane_compact): offline and
    streamed best paths, partial hypotheses and final hypotheses unchanged;
    history shrinks."""
    from paper_2311_04996_b200 import BatcherConfig, Chunk, DecoderConfig, DecodeState, StreamPool, best_path, synth

    s = _system(num_units=30, num_words=50, order=2, seed=2)
    utts = synth.planted_utterances(s, 4, 80, seed=8, gap=4.0, noise=1.0)
    cfg = DecoderConfig(beam=14.0, max_active=500)
    for u in utts:
        a, b = DecodeState(s.graph, cfg, search=search), DecodeState(s.graph, cfg, search=search)
        for i in range(0, len(u), 10):
            a.advance_frames(u[i:i + 10])
            b.advance_frames(u[i:i + 10])
            before = len([r for fr in b.history_records() for r in fr])
            kept = b.compact_history()
            assert kept <= before
            assert best_path(a) == best_path(b)
        assert sum(len(fr) for fr in b.history_records()) < sum(len(fr) for fr in a.history_records())
    # streams with collection every 2 chunks == streams without
    finals = []
    for gc in (None, 2):
        pool = StreamPool(s.graph, cfg, BatcherConfig(max_batch=3), gc_every=gc, search=search)
        sids = [pool.create_stream() for _ in utts]
        partial = []
        for sid, u in zip(sids, utts):
            for i in range(0, len(u), 9):
                pool.push_chunk(Chunk(sid, u[i:i + 9], is_last=i + 9 >= len(u)))
        while pool.ready_streams():
            partial.extend(pool.step())
        finals.append((pool.drain(), partial))
    (f0, p0), (f1, p1) = finals
    assert f0 == f1 and p0 == p1


def test_ragged_wide_nan_and_extreme_configs_match_oracle(oracle_mod):
    """Edge cases in one launch each: ragged utterance lengths, frames wider
    than the shared-memory row (log-likelihoods read from global memory),
    NaN log-likelihoods (dropped like the reference's `nc < inf` test,
    _kernel.pyx:253), f64 input, and extreme beam / max_active."""
    from paper_2311_04996_b200 import DecodeFailure, DecoderConfig, decode_batch, synth

    s = _system(num_units=12, num_words=30, order=2, seed=6, min_pron=1, max_pron=4)
    rng = np.random.default_rng(1)
    base = synth.planted_utterances(s, 6, 50, seed=4, gap=4.0, noise=1.0)
    ragged = [u[: int(rng.integers(1, 50))] for u in base]
    wide = [np.concatenate([u, rng.normal(-9.0, 1.0, size=(len(u), 5000 - u.shape[1]))], axis=1) for u in base[:3]]
    nanu = base[3].copy()
    nanu[5, :4] = np.nan
    cases = [(ragged, DecoderConfig(beam=12.0, max_active=200)),
             (wide, DecoderConfig(beam=12.0, max_active=200)),
             ([nanu], DecoderConfig(beam=12.0, max_active=200)),
             (base[:3], DecoderConfig(beam=1e-6, max_active=1)),
             (base[:3], DecoderConfig(beam=1e9, max_active=1_000_000))]
    for utts, cfg in cases:
        got = decode_batch(s.graph, cfg, utts)
        for u, h in zip(utts, got):
            try:
                want = oracle_mod.decode_utterance(s.graph, cfg, np.asarray(u, np.float64))
            except oracle_mod.OracleError:
                assert isinstance(h, DecodeFailure)
                continue
            assert (h.words, h.total_cost, h.frame_count) == want


def test_long_utterance_history_pages(oracle_mod):
    """3000 frames in 7 chunks of one channel: history spans several 64K-record
    pages and the frame-start array regrows; best path == oracle."""
    from paper_2311_04996_b200 import DecoderConfig, DecodeState, best_path, synth

    s = _system(num_units=12, num_words=30, order=2, seed=6, min_pron=1, max_pron=4)
    u = synth.planted_utterances(s, 1, 3000, seed=5, gap=3.0, noise=1.0)[0]
    cfg = DecoderConfig(beam=14.0, max_active=2000)
    ch = DecodeState(s.graph, cfg)
    for i in range(0, len(u), 450):
        ch.advance_frames(u[i:i + 450])
    oc = oracle_mod.OracleChannel.from_config(s.graph, cfg)
    oc.advance_frames(u)
    h = best_path(ch)
    assert (h.words, h.total_cost, h.frame_count) == oc.best_path()
    assert sum(len(f) for f in ch.history_records()) > 65536


# ------------------------------------------------ BASELINE configs 3 and 5 --


@pytest.fixture(scope="module")
def c3_graph(tmp_path_factory):
    """BASELINE config 3's 4-gram TLG (16.5 M states, 52.3 M arcs) built once,
    written as a .ctwg and loaded back through the memory-mapped loader."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench

    from paper_2311_04996_b200 import graphio

    s = bench.system(False, "c3")
    p = graphio.save_graph(s.graph, tmp_path_factory.mktemp("c3") / "c3.ctwg")
    return s, graphio.load_graph(p)


@pytest.mark.parametrize("search", ["exact", "fast"])
def test_c3_4gram_matches_oracle(oracle_mod, c3_graph, search):
    """Three Conformer-shaped utterances x 60 frames on the C3 graph (deep
    backoff chains, 52 M arcs) at the bench configuration: words and cost ==
    the CPU oracle; the exact mode also reproduces every record."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench

    from paper_2311_04996_b200 import DecoderConfig, DecodeState, best_path, decode_batch

    s, fg = c3_graph
    assert fg.num_arcs == s.graph.num_arcs > 50_000_000
    utts = bench.workload(s, 3, 60, 0)
    cfg = DecoderConfig(beam=bench.BEAM, max_active=bench.MAX_ACTIVE)
    got = decode_batch(fg, cfg, utts, search=search)
    for u, h in zip(utts, got):
        ow, oc, ofc = oracle_mod.decode_utterance(fg, cfg, u.astype(np.float64))
        assert h.words == ow and h.frame_count == ofc
        assert math.isclose(h.total_cost, oc, rel_tol=COST_RTOL)
        if search == "exact":
            assert h.total_cost == oc
    if search == "exact":
        ch = DecodeState(fg, cfg)
        ch.advance_frames(utts[0])
        oc = oracle_mod.OracleChannel.from_config(fg, cfg)
        oc.advance_frames(utts[0].astype(np.float64))
        assert_history_equivalent(ch.history_records(), oc.history_records(), exact_prev=False)


@pytest.mark.parametrize("search", ["exact", "fast"])
def test_c5_boosted_matches_oracle(oracle_mod, search):
    """BASELINE config 5: the C2 graph with a 100-word boost table per
    utterance (magnitudes U(0.5, 8.5)), 4 utterances x 60 frames."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench

    from paper_2311_04996_b200 import DecoderConfig, decode_batch

    s = bench.system(False, "c2")
    utts = bench.workload(s, 4, 60, 0)
    boosts = bench.boost_tables(s, 4, 0)
    cfg = DecoderConfig(beam=bench.BEAM, max_active=bench.MAX_ACTIVE)
    got = decode_batch(s.graph, cfg, utts, boost=boosts, search=search)
    for u, b, h in zip(utts, boosts, got):
        ow, oc, ofc = oracle_mod.decode_utterance(s.graph, cfg, u.astype(np.float64), boost=b)
        assert h.words == ow and h.frame_count == ofc
        assert math.isclose(h.total_cost, oc, rel_tol=COST_RTOL)
        if search == "exact":
            assert h.total_cost == oc


@pytest.mark.parametrize("search", ["exact", "fast"])
def test_stream_partials_equal_offline_prefix_decodes(search):
    """Every partial hypothesis StreamPool.step() returns (the best path
    computed behind the chunk's frame kernel in the same call) equals the
    offline decode of the same utterance prefix."""
    from paper_2311_04996_b200 import BatcherConfig, Chunk, DecoderConfig, StreamPool, decode_batch, synth

    s = _system(num_units=30, num_words=50, order=2, seed=2)
    utts = synth.planted_utterances(s, 4, 40, seed=8)
    cfg = DecoderConfig(beam=14.0, max_active=500)
    pool = StreamPool(s.graph, cfg, BatcherConfig(max_batch=4), search=search)
    sids = [pool.create_stream() for _ in utts]
    seen = {sid: 0 for sid in sids}
    partials = []
    for i in range(0, 40, 7):
        for sid, u in zip(sids, utts):
            pool.push_chunk(Chunk(sid, u[i:i + 7], is_last=i + 7 >= 40))
        for sid, h in pool.step():
            seen[sid] += 1
            partials.append((sids.index(sid), h))
    for k, h in partials:
        want = decode_batch(s.graph, cfg, [utts[k][:h.frame_count]], search=search)[0]
        assert h == want
    assert len(partials) == 4 * 6


@pytest.mark.parametrize("search", ["exact", "fast"])
def test_stream_step_graph_equals_stream_launches(monkeypatch, search):
    """A streaming step's first round runs as one CUDA graph launch (uploads,
    frame kernel, partial best paths, result copies). The graph path is the
    one taken, and its partial hypotheses equal those of plain stream
    launches (CTW_NO_GRAPH=1), chunk for chunk."""
    from paper_2311_04996_b200 import BatcherConfig, Chunk, DecoderConfig, StreamPool, synth

    s = _system(num_units=30, num_words=50, order=2, seed=2)
    utts = synth.planted_utterances(s, 5, 48, seed=3)
    cfg = DecoderConfig(beam=14.0, max_active=500)
    out = {}
    for mode in ("graph", "plain"):
        if mode == "plain":
            monkeypatch.setenv("CTW_NO_GRAPH", "1")
        pool = StreamPool(s.graph, cfg, BatcherConfig(max_batch=5), search=search)
        lp = s.graph.device_graph(0).pool(cfg, s.graph.num_states, search)
        g0 = lp.graph_info()
        sids = [pool.create_stream() for _ in utts]
        got = []
        for i in range(0, 48, 6):
            for sid, u in zip(sids, utts):
                pool.push_chunk(Chunk(sid, u[i:i + 6], is_last=i + 6 >= 48))
            got.append(sorted((sids.index(sid), h.words, h.total_cost, h.frame_count) for sid, h in pool.step()))
        g1 = lp.graph_info()
        out[mode] = (got, g1["graph_launches"] - g0["graph_launches"])
        pool.close()
    assert not lp.graph_info()["graphs_off"]
    assert out["graph"][1] >= 6 and out["plain"][1] == 0
    assert out["graph"][0] == out["plain"][0]


@pytest.mark.parametrize("chunk", [1, 5])
def test_stream_partials_with_best_path_cache(chunk):
    """Streaming partial hypotheses come from k_best_path with the per-lane
    best-path cache (the walk stops where it meets the previous step's best
    path and copies that prefix's words). On a random graph whose epsilon
    and emitting arcs both carry output labels (multi-label records), every
    partial equals the offline decode of the same prefix (fresh lanes: a
    full walk), with 1-frame chunks that reuse the cache on every step."""
    from paper_2311_04996_b200 import BatcherConfig, Chunk, DecoderConfig, FlatGraph, StreamPool, decode_batch

    rng = np.random.default_rng(11)
    S, V, W = 60, 6, 25
    src, il, ol, w, ns = [], [], [], [], []
    for s_ in range(S):
        for _ in range(int(rng.integers(1, 4))):  # emitting arcs
            src.append(s_); il.append(int(rng.integers(1, V + 1)))
            ol.append(int(rng.integers(1, W + 1)) if rng.random() < 0.4 else 0)
            w.append(float(rng.uniform(0.0, 2.0))); ns.append(int(rng.integers(0, S)))
        if rng.random() < 0.5:  # a labelled or unlabelled epsilon arc to a later state
            src.append(s_); il.append(0); ol.append(int(rng.integers(1, W + 1)) if rng.random() < 0.5 else 0)
            w.append(float(rng.uniform(0.1, 1.0))); ns.append(int(rng.integers(s_ + 1, S + 1)) % S if s_ + 1 < S else 0)
    final = np.where(rng.random(S) < 0.3, rng.uniform(0, 1, S), np.inf)
    fg = FlatGraph.from_arrays(S, 0, src, il, ol, w, ns, final)
    utts = [rng.normal(-2.0, 1.0, size=(60, V)) for _ in range(3)]
    cfg = DecoderConfig(beam=8.0, max_active=200)
    pool = StreamPool(fg, cfg, BatcherConfig(max_batch=3), search="exact")
    sids = [pool.create_stream() for _ in utts]
    partials = []
    for i in range(0, 60, chunk):
        for sid, u in zip(sids, utts):
            pool.push_chunk(Chunk(sid, u[i:i + chunk], is_last=i + chunk >= 60))
        partials += [(sids.index(sid), h) for sid, h in pool.step()]
    pool.close()
    multi = 0
    for k, h in partials:
        want = decode_batch(fg, cfg, [utts[k][:h.frame_count]])[0]
        assert h == want
        multi += len(h.words) > 1
    assert multi > 10
