"""Per-phase clock64 cycles of k_lattice_idx (instrumented build from tools/lat_mkprof.py) on 64 C2 utterances."""
import ctypes as C, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch, bench
from paper_2311_04996_b200 import DecoderConfig, decode_lattices, _lib
s = bench.system(False, "c2")
ll = torch.from_numpy(bench.workload(s, 64, 250, 0)).cuda()
cfg = DecoderConfig(beam=bench.BEAM, max_active=bench.MAX_ACTIVE)
lib = _lib.load()
buf = (C.c_ulonglong * 8)()
for it in range(3):
    decode_lattices(s.graph, cfg, ll, lattice_beam=6.0, search="fast")
    lib.ctw_latprof(buf)
    n = buf[5]
    print("ctas", n, "per CTA-layer cycles: map-clear/ac", buf[0] / n / 250, "map", buf[1] / n / 250, "src+scan", buf[2] / n / 250, "items", buf[3] / n / 250, "cl.sync", buf[4] / n / 250)
