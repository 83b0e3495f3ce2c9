"""Tiny racecheck case for the 64-register wide build: a 2-lane launch
(16 x 1024-thread CTAs per lane, one CTA per SM) in both search modes."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2311_04996_b200 import DecoderConfig, decode_batch, synth  # noqa: E402

s = synth.build_system(synth.SystemSpec(num_units=129, blank_id=128, num_words=200, order=3, seed=5, min_pron=1,
                                        max_pron=4, followers=12))
utts = list(synth.conformer_logprobs(s, 2, 4, seed=1, delta=5.0, sigma=1.5, dtype=np.float32))
cfg = DecoderConfig(beam=14.0, max_active=300)
for search in ("fast", "exact"):
    print(search, [h.words[:5] for h in decode_batch(s.graph, cfg, utts, search=search)])
