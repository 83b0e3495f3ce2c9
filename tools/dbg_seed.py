"""Debug: replay test_random_systems_history_identical_to_oracle[seed] and
print the first frame whose (tie-insensitive) records differ from the oracle."""
import sys
sys.path.insert(0, "oracle"); sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import oracle as orc
from conftest import history_signature
from paper_2311_04996_b200 import DecoderConfig, DecodeState, synth

seed = int(sys.argv[1])
spec = dict(num_units=4 + 3 * seed, num_words=10 + 7 * seed, order=1 + seed % 3, seed=seed, min_pron=1, max_pron=5)
s = synth.build_system(synth.SystemSpec(**spec))
rng = np.random.default_rng(seed)
frames = rng.normal(-3.0, 2.5, size=(60, spec["num_units"])) if seed % 2 else synth.planted_utterances(s, 1, 60, seed=seed)[0]
cfg = DecoderConfig(beam=[4.0, 9.0, 17.0, 1e9][seed % 4], max_active=[7, 60, 10_000, 300][seed % 4])
step = [60, 1, 7, 13][seed % 4]
for trial in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    ch = DecodeState(s.graph, cfg)
    oc = orc.OracleChannel.from_config(s.graph, cfg)
    for i in range(0, 60, step):
        ch.advance_frames(frames[i:i + step]); oc.advance_frames(frames[i:i + step])
    g, w = ch.history_records(), oc.history_records()
    sg, sw = history_signature(g), history_signature(w)
    bad = [f for f in range(len(sw)) if f >= len(sg) or sg[f] != sw[f]]
    print("trial", trial, "frames", len(g), len(w), "bad frames", bad[:10])
    if bad:
        f = bad[0]
        A = set(sg[f]); B = set(sw[f])
        print(" frame", f, "n", len(sg[f]), len(sw[f]))
        for r in sorted(A - B)[:8]: print("  gpu only", r[:3], len(r[3]))
        for r in sorted(B - A)[:8]: print("  ora only", r[:3], len(r[3]))
