"""Debug helper: GPU history for test_random_systems_history_identical_to_oracle[seed]."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT)]
from paper_2311_04996_b200 import DecoderConfig, DecodeState, synth

seed = int(sys.argv[1])
spec = dict(num_units=4 + 3 * seed, num_words=10 + 7 * seed, order=1 + seed % 3, seed=seed, min_pron=1, max_pron=5)
s = synth.build_system(synth.SystemSpec(**spec))
rng = np.random.default_rng(seed)
frames = rng.normal(-3.0, 2.5, size=(60, spec["num_units"])) if seed % 2 else synth.planted_utterances(s, 1, 60, seed=seed)[0]
cfg = DecoderConfig(beam=[4.0, 9.0, 17.0, 1e9][seed % 4], max_active=[7, 60, 10_000, 300][seed % 4])
ch = DecodeState(s.graph, cfg)
step = [60, 1, 7, 13][seed % 4]
for i in range(0, 60, step):
    ch.advance_frames(frames[i:i + step])
e = ch._export()
np.savez(ROOT / "gpurun_out" / f"rand_hist_{seed}.npz", frames=frames, **e)
print("ok", len(e["rec_state"]))
