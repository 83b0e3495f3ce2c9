"""Arrival-driven streaming simulation with measured service times.

Restates the reference's `stream-sim` scheduler (pkg/src/ctcwfst/cli.py:209-297)
so GPU and CPU stream pools are driven by the SAME virtual-time arrival
process: stream k submits one chunk every 1/rate seconds, streams staggered
uniformly inside that period; the server launches a batch as soon as it is free
and either max_batch streams are ready or the oldest waiting chunk has waited
max_wait_ms; the service time of a batch is the measured wall time of
`pool.step()`. Each chunk yields a (compute_ms, queue_ms) sample, aggregated
with the reference's convention (queueing.py:110-126: p-quantile =
sorted[ceil(q n) - 1]).

Works with any StreamPool exposing create_stream / push_chunk / step / drain
(ours or the reference's) -- `chunk_cls` is the matching Chunk type.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np


@dataclass
class StreamResult:
    samples: list  # (compute_ms, queue_ms) per chunk
    finals: dict   # stream id -> final Hypothesis
    server_busy_s: float
    audio_s: float
    steps: int

    def stats(self) -> dict:
        totals = sorted(c + q for c, q in self.samples)
        n = len(totals)

        def pct(q):
            return totals[max(0, math.ceil(q * n) - 1)]

        return {
            "chunks": n,
            "p50_total_ms": pct(0.50),
            "p99_total_ms": pct(0.99),
            "avg_total_ms": math.fsum(totals) / n,
            "avg_compute_ms": math.fsum(c for c, _ in self.samples) / n,
            "avg_queue_ms": math.fsum(q for _, q in self.samples) / n,
            "steps": self.steps,
            "rtfx": self.audio_s / self.server_busy_s if self.server_busy_s > 0 else 0.0,
        }


def simulate(pool, chunk_cls, utterances, chunk_frames: int = 12, rate: float = 2.0, max_batch: int = 8,
             max_wait_ms: float = 0.0, frame_s: float = 0.04, sync=None) -> StreamResult:
    """Drive `pool` with one stream per utterance ((frames, V) arrays)."""
    n = len(utterances)
    sids = [pool.create_stream() for _ in range(n)]
    period = 1.0 / rate
    arrivals = []  # (time, stream index, chunk)
    total_frames = 0
    for k, mat in enumerate(utterances):
        total_frames += mat.shape[0]
        n_chunks = max(1, math.ceil(mat.shape[0] / chunk_frames))
        for i in range(n_chunks):
            c = chunk_cls(stream_id=sids[k], frames=mat[i * chunk_frames:(i + 1) * chunk_frames],
                          is_last=(i == n_chunks - 1))
            arrivals.append((k * period / n + i * period, k, c))
    arrivals.sort(key=lambda a: (a[0], a[1]))
    k_of_sid = {s: k for k, s in enumerate(sids)}
    max_wait = max_wait_ms / 1e3
    samples = []
    server_free = 0.0
    busy = 0.0
    idx = 0
    steps = 0
    waiting: dict = {}  # (arrival time, stream index) -> None, insertion (= FIFO) order
    arrival_of: dict = {k: [] for k in range(n)}

    def admit(until):
        nonlocal idx
        while idx < len(arrivals) and arrivals[idx][0] <= until:
            t, k, c = arrivals[idx]
            pool.push_chunk(c)
            waiting[(t, k)] = None
            arrival_of[k].append(t)
            idx += 1

    while idx < len(arrivals) or waiting:
        if not waiting:
            admit(arrivals[idx][0])
            continue
        oldest = next(iter(waiting))[0]
        t0 = max(server_free, oldest)
        admit(t0)
        ready = len({k for _, k in waiting})
        if ready >= max_batch or max_wait <= 0.0:
            launch = t0  # with no batching wait the server starts as soon as it is free
        else:
            fill = math.inf
            seen = {k for _, k in waiting}
            for j in range(idx, len(arrivals)):
                seen.add(arrivals[j][1])
                if len(seen) >= max_batch:
                    fill = arrivals[j][0]
                    break
            launch = max(t0, min(oldest + max_wait, fill))
        admit(launch)
        t_start = time.perf_counter()
        advanced = pool.step()
        if sync is not None:
            sync()
        service = time.perf_counter() - t_start
        steps += 1
        busy += service
        for sid, _ in advanced:
            k = k_of_sid[sid]
            a = arrival_of[k].pop(0)
            del waiting[(a, k)]
            samples.append((service * 1e3, (launch - a) * 1e3))
        server_free = launch + service
    finals = pool.drain()
    return StreamResult(samples=samples, finals={k_of_sid[s]: h for s, h in finals.items()},
                        server_busy_s=busy, audio_s=total_frames * frame_s, steps=steps)
