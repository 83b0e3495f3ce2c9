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
