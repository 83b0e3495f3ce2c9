"""Lattice of the first N C2 bench utterances: arcs / n-best per utterance
(run with CTW_LAT_RANKS=1 and =8 to compare the cluster split)."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2311_04996_b200 import DecoderConfig, decode_lattices  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
s = bench.system(False, "c2")
ll = torch.from_numpy(bench.workload(s, n, 250, 0)).cuda()
cfg = DecoderConfig(beam=bench.BEAM, max_active=bench.MAX_ACTIVE)
lats = decode_lattices(s.graph, cfg, ll, lattice_beam=6.0)
out = [(lat.status, lat.num_arcs, len(lat.nbest(3)), round(lat.best_cost, 6)) for lat in lats]
json.dump(out, open(f"gpurun_out/diag_lat_{os.environ.get('CTW_LAT_RANKS', 'auto')}.json", "w"))
print(os.environ.get("CTW_LAT_RANKS"), [o for o in out if o[2] == 0][:5], sum(o[1] for o in out))
