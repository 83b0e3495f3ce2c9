"""Fast vs exact on the first 64 C2 bench utterances: words/costs, and the
lattice 1-best against the decode best path (diagnostics)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2311_04996_b200 import DecoderConfig, decode_batch, decode_lattices  # noqa: E402

s = bench.system(False, "c2")
ll = torch.from_numpy(bench.workload(s, 64, 250, 0)).cuda()
cfg = DecoderConfig(beam=bench.BEAM, max_active=bench.MAX_ACTIVE)
ex = decode_batch(s.graph, cfg, ll, search="exact")
fa = decode_batch(s.graph, cfg, ll, search="fast")
print("words equal", sum(a.words == b.words for a, b in zip(ex, fa)), "max cost diff",
      max(abs(a.total_cost - b.total_cost) for a, b in zip(ex, fa)))
for mode in ("exact", "fast"):
    lats = decode_lattices(s.graph, cfg, ll, lattice_beam=6.0, search=mode)
    for i, lat in enumerate(lats):
        nb = lat.nbest(3)
        if nb[0].words != lat.best_path.words:
            print(mode, i, "best", lat.best_path.total_cost, lat.best_path.words[:8], "| nb:",
                  [(h.total_cost, h.words[:8]) for h in nb])
