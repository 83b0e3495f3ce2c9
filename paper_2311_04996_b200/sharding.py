"""Utterance sharding across GPUs (BASELINE config 3).

Utterances are independent, so multi-GPU decoding is pure data parallelism:
every GPU holds its own graph replica and lane set, each decodes its shard,
and hypotheses are gathered on the host into input order -- exactly the
reference's ``decode_batch`` contract (decoder.py:436-463: input order kept,
per-index DecodeFailure), with no collective on the decode path.

Two drivers:
* ``decode_batch_devices`` -- one process, one host thread per GPU (the
  C-ABI releases the GIL, so the threads' launches overlap).
* ``decode_batch_distributed`` -- one process per GPU under
  ``torch.distributed`` (torchrun); each rank decodes its shard on its local
  GPU and the host-side results are exchanged with ``all_gather_object``
  (plumbing, not data path).

Shards are balanced by longest-processing-time on frame counts (decode time is
linear in frames); equal lengths degrade to round robin.
"""

from __future__ import annotations

import heapq
from concurrent.futures import ThreadPoolExecutor
from typing import Callable, Sequence

import numpy as np


def frame_counts(utterances: Sequence) -> list[int]:
    return [int(np.shape(u)[0]) if np.ndim(u) >= 1 else 0 for u in utterances]


def shard_lpt(frames: Sequence[int], world: int) -> list[list[int]]:
    """Longest-processing-time partition of utterance indices over `world`
    shards; each shard's indices are returned in ascending order. Ties are
    broken by index, so the partition is deterministic on every rank."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(frames)), key=lambda i: (-frames[i], i))
    heap = [(0, r) for r in range(world)]
    shards: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        shards[r].append(i)
        heapq.heappush(heap, (load + frames[i], r))
    return [sorted(s) for s in shards]


def _merge(n: int, shards: list[list[int]], parts: list[list]) -> list:
    out: list = [None] * n
    for idx, res in zip(shards, parts):
        for i, r in zip(idx, res):
            out[i] = _reindex(r, i)
    return out


def _reindex(r, i):
    """Shard-local DecodeFailure.index -> global index."""
    from .decoder import DecodeFailure

    if isinstance(r, DecodeFailure) and r.index != i:
        return DecodeFailure(index=i, error=r.error)
    return r


def decode_batch_devices(graph, config, utterances: Sequence, devices: Sequence[int], boost=None,
                         decode_fn: Callable | None = None, **kw) -> list:
    """Decode on several GPUs from one process: shard, one host thread per
    device, gather in input order."""
    from .decoder import decode_batch, flatten

    fn = decode_fn or decode_batch
    fg = flatten(graph)
    n = len(utterances)
    shards = shard_lpt(frame_counts(utterances), len(devices))
    per_utt = isinstance(boost, (list, tuple))

    def run(k):
        idx = shards[k]
        if not idx:
            return []
        b = [boost[i] for i in idx] if per_utt else boost
        return fn(fg, config, [utterances[i] for i in idx], boost=b, device=devices[k], **kw)

    with ThreadPoolExecutor(max_workers=len(devices)) as pool:
        parts = list(pool.map(run, range(len(devices))))
    return _merge(n, shards, parts)


def decode_batch_distributed(graph, config, utterances: Sequence, boost=None, group=None,
                             decode_fn: Callable | None = None, device: int | None = None, **kw) -> list:
    """Decode under torch.distributed: every rank passes the SAME utterance
    list, decodes its LPT shard on its local device and receives the full
    result list (input order)."""
    import torch.distributed as dist

    from .decoder import decode_batch, flatten

    fn = decode_fn or decode_batch
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = len(utterances)
    shards = shard_lpt(frame_counts(utterances), world)
    idx = shards[rank]
    per_utt = isinstance(boost, (list, tuple))
    b = [boost[i] for i in idx] if per_utt else boost
    mine = fn(flatten(graph), config, [utterances[i] for i in idx], boost=b, device=device, **kw) if idx else []
    parts: list = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    return _merge(n, shards, parts)
