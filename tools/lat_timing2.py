"""Wall-time split of decode_lattices (no profiler): the C call vs Python."""
import cProfile
import pstats
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
for _ in range(2):
    decode_lattices(s.graph, cfg, ll, lattice_beam=6.0, search="fast")
torch.cuda.synchronize(); t0 = time.perf_counter()
decode_batch(s.graph, cfg, ll, search="fast")
torch.cuda.synchronize(); t1 = time.perf_counter()
decode_lattices(s.graph, cfg, ll, lattice_beam=6.0, search="fast")
torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"n={n} decode {t1 - t0:.4f} decode+lattice {t2 - t1:.4f} lattice stage {t2 - t1 - (t1 - t0):.4f}")
pr = cProfile.Profile()
pr.enable()
decode_lattices(s.graph, cfg, ll, lattice_beam=6.0, search="fast")
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
