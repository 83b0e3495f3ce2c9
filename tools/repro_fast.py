"""Small fast-mode decode (random system 0 of test_fast_mode) for sanitizer runs."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_04996_b200 import DecoderConfig, DecodeState, best_path, synth  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
spec = dict(num_units=4 + 3 * seed, num_words=10 + 7 * seed, order=1 + seed % 3, seed=seed, min_pron=1, max_pron=5)
s = synth.build_system(synth.SystemSpec(**spec))
rng = np.random.default_rng(seed)
frames = rng.normal(-3.0, 2.5, size=(60, spec["num_units"])) if seed % 2 else synth.planted_utterances(s, 1, 60, seed=seed)[0]
cfg = DecoderConfig(beam=[4.0, 9.0, 17.0, 1e9][seed % 4], max_active=[7, 60, 10_000, 300][seed % 4])
ch = DecodeState(s.graph, cfg, search="fast")
step = [60, 1, 7, 13][seed % 4]
for i in range(0, 60, step):
    ch.advance_frames(frames[i:i + step])
print(best_path(ch), ch._pool.profile())
