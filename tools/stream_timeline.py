"""GPU timeline of streaming steps (torch.profiler / CUPTI): what a
StreamPool.step() of a few C2 streams puts on the device besides the frame
kernel. Diagnostics only.  python tools/stream_timeline.py [streams] [steps]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2311_04996_b200 import BatcherConfig, Chunk, DecoderConfig, StreamPool  # noqa: E402

ns = int(sys.argv[1]) if len(sys.argv) > 1 else 6
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
s = bench.system(False, "c2")
utts = list(bench.workload(s, ns, 12 * (2 * steps + 12), 7000))
pool = StreamPool(s.graph, DecoderConfig(beam=bench.BEAM, max_active=bench.MAX_ACTIVE),
                  BatcherConfig(max_batch=ns), device=0, search="fast")
sids = [pool.create_stream() for _ in range(ns)]


def step(i):
    for k, sid in enumerate(sids):
        pool.push_chunk(Chunk(stream_id=sid, frames=utts[k][12 * i:12 * (i + 1)], is_last=False))
    pool.step()


for i in range(10):
    step(i)
torch.cuda.synchronize()
import time  # noqa: E402

t0 = time.perf_counter()
for i in range(10, 10 + steps):
    step(i)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / steps
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    for i in range(10 + steps, 10 + 2 * steps):
        step(i)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
tot = {}
for e in ev:
    k = e.name[:50]
    tot.setdefault(k, [0, 0.0])
    tot[k][0] += 1
    tot[k][1] += e.time_range.elapsed_us()
print(f"streams {ns}: wall per step {wall * 1e3:.3f} ms (no profiler)")
for k, (c, us) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"  {k:50s} {c / steps:5.1f}/step {us / steps:8.1f} us/step")
# device span per step and idle gaps inside it
span = (ev[-1].time_range.end - ev[0].time_range.start) / steps
busy = sum(e.time_range.elapsed_us() for e in ev) / steps
print(f"device span/step {span:.1f} us, busy {busy:.1f} us")
