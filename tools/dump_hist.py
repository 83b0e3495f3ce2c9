"""Debug helper: dump GPU histories for golden cases to gpurun_out/hist_*.npz."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests"), str(ROOT / "oracle")]
from conftest import GoldenGraph, golden_chunks, golden_names, load_golden
from paper_2311_04996_b200 import DecodeError, DecodeState, DecoderConfig, flatten

for name in sys.argv[1:] or golden_names():
    d = load_golden(name)
    cfg = DecoderConfig(beam=d["beam"], max_active=d["max_active"], acoustic_scale=d["acoustic_scale"],
                        nonemitting_relax_epsilon=d["relax_eps"],
                        max_nonemitting_iters=None if d["max_ne_iters"] < 0 else d["max_ne_iters"])
    ch = DecodeState(flatten(GoldenGraph(d)), cfg)
    b = d["boost"] if d["has_boost"] else None
    if b is not None:
        if d["boost_poke"]: ch.boost = b
        else: ch.set_boost(b)
    err = ""
    for c in golden_chunks(d):
        try:
            ch.advance_frames(c)
        except DecodeError as e:
            err = str(e); break
    e = ch._export()
    np.savez(ROOT / "gpurun_out" / f"hist_{name}.npz", err=err, **e)
    print(name, err, len(e["rec_state"]))
