"""Lattice leg split: decode, decode+lattice wall time, and the k_lattice
kernel time (CUDA events around ctw_lane_lattice's launches, from ncu-free
timing: torch profiler not needed -- the library's own stats)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2311_04996_b200 import DecoderConfig, decode_batch, decode_lattices  # noqa: E402

s = bench.system(False, "c2")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ll = torch.from_numpy(bench.workload(s, n, 250, 0)).cuda()
cfg = DecoderConfig(beam=bench.BEAM, max_active=bench.MAX_ACTIVE)
decode_lattices(s.graph, cfg, ll, lattice_beam=6.0, search="fast")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    decode_batch(s.graph, cfg, ll, search="fast")
    torch.cuda.synchronize(); t1 = time.perf_counter()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        lats = decode_lattices(s.graph, cfg, ll, lattice_beam=6.0, search="fast")
    torch.cuda.synchronize(); t2 = time.perf_counter()
    ev = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name.split("(")[0][-40:]
            ev[k] = ev.get(k, 0.0) + e.device_time_total / 1e3
    print(f"n={n} decode {t1 - t0:.4f}s  decode+lattice {t2 - t1:.4f}s  kernels(ms): "
          + ", ".join(f"{k}={v:.1f}" for k, v in sorted(ev.items(), key=lambda x: -x[1])[:6]))
