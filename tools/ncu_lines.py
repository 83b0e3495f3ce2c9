"""Aggregate ncu warp-stall samples per CUDA source line.

    ncu -i report.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
agg, text, cur = {}, {}, None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0].strip():
        cur = int(r[0])
        text[cur] = r[1]
    try:
        v = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        v = 0.0
    if cur is not None:
        agg[cur] = agg.get(cur, 0.0) + v
tot = sum(agg.values()) or 1
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}%  {ln:5d}  {text.get(ln, '').strip()[:100]}")
