"""Arc-level diff of lattices built with 1 vs 8 CTAs per lane (diagnostics)."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_04996_b200 import DecoderConfig, decode_lattices, synth  # noqa: E402

s = synth.build_system(synth.SystemSpec(num_units=129, blank_id=128, num_words=300, order=3, seed=5, min_pron=1,
                                        max_pron=4, followers=15))
utts = list(synth.conformer_logprobs(s, 12, 80, seed=2, delta=5.0, sigma=1.5, dtype=np.float32))
cfg = DecoderConfig(beam=14.0, max_active=500)
out = {}
for r in ("1", "8", "1"):
    os.environ["CTW_LAT_RANKS"] = r
    out.setdefault(r, []).append(decode_lattices(s.graph, cfg, utts, lattice_beam=5.0))
for i in range(len(utts)):
    a, b, c = out["1"][0][i], out["8"][0][i], out["1"][1][i]
    A = sorted(zip(a.frame.tolist(), a.src_state.tolist(), a.dst_state.tolist(), a.weight.tolist(), a.labels))
    B = sorted(zip(b.frame.tolist(), b.src_state.tolist(), b.dst_state.tolist(), b.weight.tolist(), b.labels))
    Cc = sorted(zip(c.frame.tolist(), c.src_state.tolist(), c.dst_state.tolist(), c.weight.tolist(), c.labels))
    sa, sb = set(A), set(B)
    print(i, len(A), len(B), "1vs1 same:", A == Cc, "1vs8 same:", A == B, "only1:", sorted(sa - sb)[:3], "only8:", sorted(sb - sa)[:3])
