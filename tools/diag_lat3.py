"""Lattice work counters on the first N C2 bench utterances: closure items /
pruned items / kept arcs per layer, and the kernel's share of the stage."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2311_04996_b200 import DecoderConfig, decode_lattices  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
s = bench.system(False, "c2")
ll = torch.from_numpy(bench.workload(s, n, 250, 0)).cuda()
cfg = DecoderConfig(beam=bench.BEAM, max_active=bench.MAX_ACTIVE)
for _ in range(2):
    lats = decode_lattices(s.graph, cfg, ll, lattice_beam=6.0, search="fast")
items = np.array([x.closure_items for x in lats]) / 250
pruned = np.array([x.closure_pruned for x in lats]) / 250
arcs = np.array([x.num_arcs for x in lats]) / 250
print(f"per layer: items {items.mean():.0f} (max {items.max():.0f}) pruned {pruned.mean():.0f} arcs {arcs.mean():.1f}")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    decode_lattices(s.graph, cfg, ll, lattice_beam=6.0, search="fast")
    torch.cuda.synchronize()
for e in prof.key_averages():
    if e.device_time_total > 100:
        print(f"{e.key[:60]:60s} {e.count:4d} {e.device_time_total / 1000:.1f} ms")
