"""cProfile of the C4 streaming run (2000 streams, fast mode): host-side cost per step."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

s = bench.system(False, "c2")
bench.streaming_run(s, 2000, 4.0, 100, device=0, search="fast")
pr = cProfile.Profile()
pr.enable()
st, _, _ = bench.streaming_run(s, 2000, 4.0, 0, device=0, search="fast")
pr.disable()
print({k: st[k] for k in ("p50_total_ms", "p99_total_ms", "steps")}, st["breakdown_s"])
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
