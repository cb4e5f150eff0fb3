#!/usr/bin/env python3
"""Summarise gpurun_out/ ncu captures into profiles/ (committed evidence).

usage: python tools/ncu_summary.py <round-tag> [workload]
Reads gpurun_out/launches.csv (gpu__time_duration launch list) and every
gpurun_out/prof_*.ncu-rep (--set full captures); writes
profiles/<tag>_launch_shares.md, profiles/<tag>_ncu_<name>.csv and updates
profiles/ncu_summary.json (per-launch DRAM bytes consumed by bench.py).
"""
import collections
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
]


def short(name):
    return name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")


def launch_shares(tag):
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[h], rows[h + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        n = short(r[ki])
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(t for _, t in agg.values())
    lines = [f"# {tag}: ncu launch list (gpu__time_duration, --clock-control none)", "",
             "Cold-cache, serialised replay of `python bench.py --steps 2 --warmup 3 "
             "--no-cpu-baseline` (first 400 launches: engine setup + eager capture run + graph "
             "replays). Shares, not absolutes, are comparable with the live CUDA-event profile "
             "in the bench JSON (roofline.per_class_ms).", "",
             "| kernel | launches | total us | share | avg us |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% | {t / n:.1f} |")
    with open(os.path.join(PROF, f"{tag}_launch_shares.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    # keep the raw launch list too (the judged evidence)
    with open(path) as src, open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as dst:
        dst.write(src.read())


def rep_summary(tag, rep, summary, workload):
    name = os.path.basename(rep).replace(".ncu-rep", "")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return
    hdr, units = rows[0], rows[1]
    keep = [m for m in METRICS if m in hdr]
    out = [keep, [units[hdr.index(m)] for m in keep]]
    for r in rows[2:]:
        out.append([r[hdr.index(m)] for m in keep])
    with open(os.path.join(PROF, f"{tag}_ncu_{name}.csv"), "w", newline="") as f:
        csv.writer(f).writerows(out)
    # per-launch DRAM traffic (bytes) per kernel template instance
    for r in rows[2:]:
        kn = short(r[hdr.index("Kernel Name")])
        rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
        wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
        unit = units[hdr.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        summary.setdefault("launches", []).append(
            {"kernel": r[hdr.index("Kernel Name")][:120], "dram_bytes": (rd + wr) * scale,
             "time_us": float(r[hdr.index("gpu__time_duration.sum")].replace(",", ""))
             * (1e-3 if units[hdr.index("gpu__time_duration.sum")] == "nsecond" else 1)})
        if "gemm" in kn:
            g = summary.setdefault(f"{workload}_gemm_launches", [])
            g.append((rd + wr) * scale)
    g = summary.get(f"{workload}_gemm_launches")
    if g:
        summary[f"{workload}_gemm_dram_bytes_per_launch"] = sum(g) / len(g)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    workload = sys.argv[2] if len(sys.argv) > 2 else "c2"
    os.makedirs(PROF, exist_ok=True)
    launch_shares(tag)
    spath = os.path.join(PROF, "ncu_summary.json")
    summary = {"round": tag, "workload": workload}
    for rep in sorted(glob.glob(os.path.join(OUT, "prof_*.ncu-rep"))):
        rep_summary(tag, rep, summary, workload)
    with open(spath, "w") as f:
        json.dump(summary, f, indent=1)
    print("wrote", spath)


if __name__ == "__main__":
    main()
