"""Multi-GPU host logic on CPU: LPT sharding, input-order gather, per-index
failures, and the torch.distributed driver over gloo with world_size 2.

The decode function is injected (no GPU here); it tags each hypothesis with
the rank that produced it so the test can check the partition."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_04996_b200.decoder import DecodeFailure, DecodeError, Hypothesis
from paper_2311_04996_b200.sharding import decode_batch_devices, decode_batch_distributed, shard_lpt


def _fake_decode(tag):
    def fn(fg, cfg, utts, boost=None, device=None):
        out = []
        for k, u in enumerate(utts):
            if u.shape[0] == 0:
                out.append(DecodeFailure(index=k, error=DecodeError("no frames decoded")))
            else:
                out.append(Hypothesis(words=(int(u[0, 0]), tag if tag is not None else device),
                                      total_cost=float(u.shape[0]), frame_count=int(u.shape[0])))
        return out
    return fn


class _G:
    """Minimal FlatGraph-shaped object."""
    num_states, start = 1, 0
    off = np.zeros(2, np.int64)
    eps_end = np.zeros(1, np.int64)
    ilabel = olabel = nextstate = np.zeros(0, np.int32)
    weight = np.zeros(0)
    final = np.zeros(1)
    max_ilabel = max_olabel = 0


def _utts(n=11):
    rng = np.random.default_rng(0)
    out = []
    for i in range(n):
        f = int(rng.integers(0, 40)) if i != 3 else 0
        m = np.zeros((f, 4))
        if f:
            m[0, 0] = i
        out.append(m)
    return out


def test_lpt_balances_and_covers():
    frames = [250, 250, 10, 300, 120, 120, 5, 60]
    shards = shard_lpt(frames, 3)
    assert sorted(i for s in shards for i in s) == list(range(len(frames)))
    loads = [sum(frames[i] for i in s) for s in shards]
    assert max(loads) - min(loads) <= max(frames)
    assert shard_lpt([7] * 6, 3) == [[0, 3], [1, 4], [2, 5]]  # equal lengths: round robin
    assert shard_lpt(frames, 3) == shards  # deterministic


def test_devices_driver_keeps_input_order_and_failures():
    utts = _utts()
    got = decode_batch_devices(_G(), None, utts, devices=[0, 1, 2], decode_fn=_fake_decode(None))
    for i, (u, h) in enumerate(zip(utts, got)):
        if u.shape[0] == 0:
            assert isinstance(h, DecodeFailure) and h.index == i
        else:
            assert h.words[0] == i and h.frame_count == u.shape[0]
    assert {h.words[1] for h in got if isinstance(h, Hypothesis)} == {0, 1, 2}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        utts = _utts()
        got = decode_batch_distributed(_G(), None, utts, decode_fn=_fake_decode(rank))
        q.put((rank, [(type(h).__name__, getattr(h, "words", None), getattr(h, "index", None)) for h in got]))
    finally:
        dist.destroy_process_group()


def test_distributed_driver_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]  # every rank receives the full, identical result list
    utts = _utts()
    shards = shard_lpt([u.shape[0] for u in utts], 2)
    owner = {i: r for r, s in enumerate(shards) for i in s}
    for i, (kind, words, index) in enumerate(res[0]):
        if utts[i].shape[0] == 0:
            assert kind == "DecodeFailure" and index == i
        else:
            assert words == (i, owner[i])


def test_decode_split_halves_groups_on_device_oom(monkeypatch):
    """decode_batch's out-of-memory handling: a group that
    does not fit is halved until it does; a single utterance that cannot fit
    fails with MemoryError at its own index -- never the whole batch."""
    from paper_2311_04996_b200 import decoder as D

    calls = []

    def fake_group(fg, config, pool, utterances, idx, boost, per_utt, results, lattice_beam=None):
        calls.append(list(idx))
        if len(idx) > 2 or 5 in idx:
            raise RuntimeError("lane reset failed (-102): salloc(...): out of memory")
        for i in idx:
            results[i] = Hypothesis(words=(i,), total_cost=0.0, frame_count=1)

    monkeypatch.setattr(D, "_decode_group", fake_group)
    results = [None] * 8
    D._decode_split(None, None, None, None, list(range(8)), None, False, results, None)
    assert [type(r).__name__ for r in results] == ["Hypothesis"] * 5 + ["DecodeFailure"] + ["Hypothesis"] * 2
    assert isinstance(results[5].error, MemoryError) and results[5].index == 5
    assert all(r.words == (i,) for i, r in enumerate(results) if isinstance(r, Hypothesis))
    with pytest.raises(RuntimeError, match="boom"):
        monkeypatch.setattr(D, "_decode_group", lambda *a, **k: (_ for _ in ()).throw(RuntimeError("boom")))
        D._decode_split(None, None, None, None, [0, 1], None, False, [None, None], None)


@pytest.mark.gpu
def test_devices_driver_with_real_decoder():
    """decode_batch_devices over a (repeated) device list with the real GPU
    decoder == decode_batch, in input order, failures at their index."""
    from paper_2311_04996_b200 import DecoderConfig, decode_batch, synth

    s = synth.build_system(synth.SystemSpec(num_units=12, num_words=30, order=2, seed=3))
    utts = synth.planted_utterances(s, 9, 40, seed=5)
    utts[4] = np.zeros((0, 12))
    cfg = DecoderConfig(beam=12.0, max_active=300)
    want = decode_batch(s.graph, cfg, utts, search="fast")
    got = decode_batch_devices(s.graph, cfg, utts, devices=[0, 0, 0], search="fast")
    assert [type(x) for x in got] == [type(x) for x in want]
    for a, b in zip(got, want):
        if isinstance(b, Hypothesis):
            assert a == b
        else:
            assert a.index == b.index


def _nccl_worker(rank, world, port, out):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    from paper_2311_04996_b200 import DecoderConfig, synth

    s = synth.build_system(synth.SystemSpec(num_units=12, num_words=30, order=2, seed=3))
    utts = synth.planted_utterances(s, 7, 40, seed=6)
    cfg = DecoderConfig(beam=12.0, max_active=300)
    got = decode_batch_distributed(s.graph, cfg, utts, device=0, search="fast")
    out.put([(h.words, h.total_cost) for h in got])
    dist.destroy_process_group()


@pytest.mark.gpu
def test_distributed_driver_nccl_world_1_with_real_decoder():
    """decode_batch_distributed under a world-size-1 NCCL process group with
    the real decoder == decode_batch."""
    from paper_2311_04996_b200 import DecoderConfig, decode_batch, synth

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    p = ctx.Process(target=_nccl_worker, args=(0, 1, port, q))
    p.start()
    got = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    s = synth.build_system(synth.SystemSpec(num_units=12, num_words=30, order=2, seed=3))
    utts = synth.planted_utterances(s, 7, 40, seed=6)
    want = decode_batch(s.graph, DecoderConfig(beam=12.0, max_active=300), utts, search="fast")
    assert got == [(h.words, h.total_cost) for h in want]
