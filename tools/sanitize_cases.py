"""Small workloads for compute-sanitizer runs (memcheck / racecheck /
synccheck): every golden fixture (BASELINE config 1 and the known-answer
graphs) in both search modes, a 2-lane (wide) and a 40-lane launch, lattices
on 8-CTA clusters with both lattice kernels (closure-index build included),
streaming steps as CUDA graphs with the best-path cache, and history
compaction.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from conftest import GoldenGraph, golden_chunks, golden_names, load_golden  # noqa: E402

from paper_2311_04996_b200 import (BatcherConfig, Chunk, DecodeError, DecoderConfig, DecodeState,  # noqa: E402
                                   StreamPool, best_path, decode_batch, decode_lattices, flatten, synth)

QUICK = "--quick" in sys.argv  # racecheck: a few goldens and the 2-lane cluster launch only
RACE2 = "--race2" in sys.argv  # racecheck of the round-2 additions: tiny lattices (both kernels) and streaming
n_ok = 0
for name in ([] if RACE2 else golden_names()[:2] + ["kat_eps_olabels"] if QUICK else golden_names()):
    d = load_golden(name)
    cfg = DecoderConfig(beam=d["beam"], max_active=d["max_active"], acoustic_scale=d["acoustic_scale"],
                        nonemitting_relax_epsilon=d["relax_eps"],
                        max_nonemitting_iters=None if d["max_ne_iters"] < 0 else d["max_ne_iters"])
    for search in ("exact", "fast"):
        ch = DecodeState(flatten(GoldenGraph(d)), cfg, search=search)
        if d["has_boost"]:
            ch.set_boost(d["boost"])
        try:
            for c in golden_chunks(d):
                ch.advance_frames(c)
        except DecodeError:
            pass
        if ch.frame_count and d["frame_count"] and list(best_path(ch).words) == d["best_words"].tolist():
            n_ok += 1
print("goldens with matching words:", n_ok)

# launch shapes: a 2-lane launch runs the wide kernel (1024-thread CTAs, 16
# per lane); a 40-lane launch the full-batch shape (512-thread CTAs, 8 per
# lane); lattices on 8-CTA clusters
os.environ["CTW_LAT_RANKS"] = "8"
s = synth.build_system(synth.SystemSpec(num_units=129, blank_id=128, num_words=200, order=3, seed=5, min_pron=1,
                                        max_pron=4, followers=12))
utts = list(synth.conformer_logprobs(s, 2, 8 if QUICK else 10 if RACE2 else 30, seed=1, delta=5.0, sigma=1.5,
                                     dtype=np.float32))
cfg = DecoderConfig(beam=14.0, max_active=300)
for search in (() if RACE2 else ("exact", "fast")):
    print(search, [h.words[:5] for h in decode_batch(s.graph, cfg, utts, search=search)])
    many = list(synth.conformer_logprobs(s, 40, 6, seed=2, delta=5.0, sigma=1.5, dtype=np.float32))
    print(search, "40 lanes:", sum(len(h.words) for h in decode_batch(s.graph, cfg, many, search=search)))
if QUICK:
    sys.exit(0)
lats = decode_lattices(s.graph, cfg, utts, lattice_beam=4.0)  # indexed kernel (closure index)
print("lattice arcs", [lat.num_arcs for lat in lats])
os.environ["CTW_LAT_NOPRE"] = "1"  # the general kernel (per-item closures)
print("lattice arcs (general)", [lat.num_arcs for lat in decode_lattices(s.graph, cfg, utts, lattice_beam=4.0)])
del os.environ["CTW_LAT_NOPRE"]
# streaming: step graphs, the best-path cache (5-frame chunks: the walk stops
# at the previous step's path) and history compaction every 2 steps
pool = StreamPool(s.graph, cfg, BatcherConfig(max_batch=2), search="fast", gc_every=2)
sids = [pool.create_stream() for _ in utts]
T = utts[0].shape[0]
for i in range(0, T, 5):
    for sid, u in zip(sids, utts):
        pool.push_chunk(Chunk(sid, u[i:i + 5], is_last=i + 5 >= T))
print("stream finals", {k: v.words[:5] for k, v in pool.drain().items()})
