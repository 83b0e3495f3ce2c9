"""Summarise an ncu launch list (csv) and one --set full capture into the
profiles/ evidence files bench.py reads.

    python tools/ncu_summary.py LAUNCHES.csv FULL.ncu-rep TAG [SEARCH]

writes profiles/TAG_launches.json, profiles/TAG_full_metrics.json and
refreshes profiles/traffic.json + profiles/ncu_metrics.json (the numbers
bench.py's roofline quotes)."""

import csv
import io
import json
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"

FULL_METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_threads_per_warp_instruction",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_throughput_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum": "local_ld_sectors",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": "global_ld_sectors",
}


def _num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def launches(path):
    text = Path(path).read_text()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    per = {}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        lid = int(r[ix["ID"]])
        d = per.setdefault(lid, {"id": lid, "kernel": r[ix["Kernel Name"]].split("(")[0].replace("<unnamed>::", "").removeprefix("void ")})
        name, unit, val = r[ix["Metric Name"]], r[ix["Metric Unit"]], _num(r[ix["Metric Value"]])
        scale = {"ms": 1.0, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "nsecond": 1e-6, "s": 1e3,
                 "second": 1e3, "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}.get(unit, 1.0)
        if name == "gpu__time_duration.sum":
            d["ms"] = val * scale
        elif name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            d["dram_gb"] = d.get("dram_gb", 0.0) + val * scale
        elif name == "lts__t_sector_hit_rate.pct":
            d["l2_hit_pct"] = val
    out = sorted(per.values(), key=lambda d: d["id"])
    tot = sum(d.get("ms", 0.0) for d in out) or 1.0
    by = {}
    for d in out:
        b = by.setdefault(d["kernel"], {"launches": 0, "ms": 0.0})
        b["launches"] += 1
        b["ms"] += d.get("ms", 0.0)
    for b in by.values():
        b["share_pct"] = round(100 * b["ms"] / tot, 3)
    dec = [d for d in out if d["kernel"].startswith("k_decode_chunk")]
    big = max((d.get("ms", 0.0) for d in dec), default=0.0)
    steady = [d for d in dec if d.get("ms", 0.0) > 0.5 * big]
    ss = {"launches": len(steady),
          "mean_ms": statistics.mean(d["ms"] for d in steady) if steady else None,
          "mean_dram_gb": statistics.mean(d.get("dram_gb", 0.0) for d in steady) if steady else None,
          "mean_l2_hit_pct": statistics.mean(d.get("l2_hit_pct", 0.0) for d in steady) if steady else None}
    return {"by_kernel": by, "steady_state_decode": ss, "launches": out}


def full(path):
    raw = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
    for k, name in FULL_METRICS.items():
        if k in hdr:
            i = hdr.index(k)
            out[name] = _num(vals[i])
            if units[i]:
                out[name + "_unit"] = units[i]
    return out


def main():
    lcsv, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    search = sys.argv[4] if len(sys.argv) > 4 else "fast"  # bench.py --search of the captured runs
    L = launches(lcsv)
    L["command"] = ("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                    "lts__t_sector_hit_rate.pct --clock-control none --csv python bench.py --search " + search +
                    " --steps 1 --warmup 3 --no-cpu --streams 0 --lattice 0")
    L["note"] = ("serialised, cold-cache launch list (compare shares, not absolutes); the steady-state "
                 "k_decode_chunk launches are 512 lanes x 250 frames; short decode launches are first-call grow re-runs")
    (PROF / f"{tag}_launches.json").write_text(json.dumps(L, indent=1))
    F = full(rep)
    F["command"] = ("ncu --set full --clock-control none --import-source on -k regex:k_decode_chunk -s 6 -c 1 "
                    "python bench.py --search " + search + " --batch 512 --frames 80 --steps 1 --warmup 8 --no-cpu "
                    "--streams 0 --lattice 0")
    (PROF / f"{tag}_full_metrics.json").write_text(json.dumps(F, indent=1))
    ss = L["steady_state_decode"]
    dram = ss["mean_dram_gb"] * 1e9
    (PROF / "traffic.json").write_text(json.dumps({
        "kernel": "k_decode_chunk", "dram_bytes_per_launch": dram, "search": search, "config": "c2",
        "source": f"profiles/{tag}_launches.json: mean of the steady-state 512x250 launches "
                  "(dram__bytes_read.sum + dram__bytes_write.sum)"}, indent=1))
    (PROF / "ncu_metrics.json").write_text(json.dumps({
        "kernel": F.get("kernel"),
        "source": f"profiles/{tag}_full_metrics.json (ncu --set full, 512 lanes x 80 frames) and "
                  f"profiles/{tag}_launches.json (512 x 250 launches)",
        "dram_bytes_per_launch": dram,
        "l2_hit_pct": F.get("l2_hit_pct"), "l1_hit_pct": F.get("l1_hit_pct"),
        "achieved_occupancy_pct": F.get("achieved_occupancy_pct"),
        "active_threads_per_warp_instruction": F.get("active_threads_per_warp_instruction"),
        "issue_slots_busy_pct": F.get("issue_slots_busy_pct"),
        "dram_throughput_pct": F.get("dram_throughput_pct"),
        "local_ld_sectors": F.get("local_ld_sectors")}, indent=1))
    print(json.dumps({"by_kernel": L["by_kernel"], "steady": ss, "full": F}, indent=1))


if __name__ == "__main__":
    main()
