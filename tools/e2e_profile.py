"""Host-side cost of one C2 decode_batch call (512 x 250 frames, pinned host
input): wall time vs the frame kernel, and a cProfile of the Python side."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2311_04996_b200 import DecoderConfig, decode_batch  # noqa: E402

s = bench.system(False, "c2")
host = torch.from_numpy(bench.workload(s, 512, 250, 0)).pin_memory().numpy()
cfg = DecoderConfig(beam=bench.BEAM, max_active=bench.MAX_ACTIVE)
for _ in range(2):
    decode_batch(s.graph, cfg, host, search="fast")
lp = s.graph.device_graph(0).pool(cfg, s.graph.num_states, "fast")
for _ in range(3):
    h0 = lp.host_timing()
    k0 = lp.stats()["decode_ms"]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    decode_batch(s.graph, cfg, host, search="fast")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h1 = lp.host_timing()
    print(f"wall {1e3 * (t1 - t0):.1f} ms, frame kernel {lp.stats()['decode_ms'] - k0:.1f} ms,",
          {k: round(1e3 * (h1[k] - h0[k]), 2) for k in h1 if isinstance(h1[k], float)})
pr = cProfile.Profile()
pr.enable()
decode_batch(s.graph, cfg, host, search="fast")
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
