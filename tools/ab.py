"""A/B timing of library variants on the bench's C2 workload.

    python tools/ab.py tools/variants/lib_a.so tools/variants/lib_b.so ... [--steps 3] [--config c2]

Each variant runs in its own process (CTW_B200_LIB selects the library):
warm-up, then `steps` timed decode_batch calls (CUDA events, L2 flushed
between steps); prints RTFx, the kernel's per-lane-frame cycles and a digest
of every transcript + cost, so variants that change results stand out.
Diagnostics only (not a bench number)."""

import argparse
import hashlib
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def child(args):
    sys.path.insert(0, str(ROOT))
    import numpy as np  # noqa: F401
    import torch

    import bench
    from paper_2311_04996_b200 import DecoderConfig, decode_batch

    s = bench.system(False, args.config)
    fg = s.graph
    cfg = DecoderConfig(beam=bench.BEAM, max_active=bench.MAX_ACTIVE)
    ll = torch.from_numpy(bench.workload(s, args.batch, args.frames, 0)).cuda()
    boosts = bench.boost_tables(s, args.batch, 0) if args.config == "c5" else None
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    pool = fg.device_graph(0).pool(cfg, fg.num_states, args.search)
    for _ in range(args.warmup):
        out = decode_batch(fg, cfg, ll, device=0, boost=boosts, search=args.search)
    pool.reset_stats()
    ms = []
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = decode_batch(fg, cfg, ll, device=0, boost=boosts, search=args.search)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    h = hashlib.sha256()
    for o in out:
        h.update(repr((o.words, round(o.total_cost, 9))).encode())
    prof = pool.profile()
    st = pool.stats()
    frames = max(1, st["frames"])
    audio = args.batch * args.frames * bench.FRAME_S
    print(json.dumps({"lib": os.environ.get("CTW_B200_LIB"), "rtfx": audio / (min(ms) / 1e3),
                      "rtfx_mean": audio / (sum(ms) / len(ms) / 1e3), "ms": ms,
                      "cycles_per_lane_frame": sum(prof[k] for k in ("emit", "eps", "beam_count", "select",
                                                                    "records", "reset")) / (frames / 1),
                      "stage": {k: prof[k] / frames for k in ("emit", "eps", "beam_count", "select", "records", "r15",
                                                              "reset", "ties")},
                      "slots": prof["slots"] / frames, "eps_items": prof["eps_items"] / frames,
                      "digest": h.hexdigest()[:16]}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="*")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=512)
    ap.add_argument("--frames", type=int, default=250)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--search", default="fast")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--rounds", type=int, default=1, help="repeat the whole variant list (interleaved)")
    args = ap.parse_args()
    if args.child:
        child(args)
        return
    for _ in range(args.rounds):
        for lib in args.libs:
            env = dict(os.environ, CTW_B200_LIB=str(Path(lib).resolve()))
            cmd = [sys.executable, __file__, "--child", "--steps", str(args.steps), "--warmup", str(args.warmup),
                   "--batch", str(args.batch), "--frames", str(args.frames), "--config", args.config,
                   "--search", args.search]
            r = subprocess.run(cmd, env=env, capture_output=True, text=True)
            line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-2000:]
            print(Path(lib).name, line, flush=True)


if __name__ == "__main__":
    main()
