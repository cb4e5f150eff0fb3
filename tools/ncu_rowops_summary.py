#!/usr/bin/env python3
"""Summarise the ncu --set full captures of the C2 row kernels
(tools/gpu_rowops_profiles.sh -> gpurun_out/prof_<kernel>.ncu-rep) into
profiles/<tag>_ncu_rowops.md: duration, DRAM bytes vs the algorithmic bytes
of one launch, and the HBM fraction of the measured peak."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M, D, N_ITEMS, TASK_COLS = 24832, 1024, 256, 7
# algorithmic bytes per launch at C2 (one query: M packed rows, d_model D)
ALG = {
    "layer_norm_kernel": (4 * D * M + 2 * D * M, "read x fp32 + write LN(x) bf16"),
    "embed_ln_kernel": (4 * D * M + 2 * D * M + 4 * D * (300 + 352),
                        "write x fp32 + LN1(x) bf16; embedding tables read once"),
    "score_head_kernel": (N_ITEMS * 4 * D + TASK_COLS * 4 * D + N_ITEMS * 6 * 8,
                          "last-row x fp32 + head weights + scores f64"),
    "topk_scores_kernel": (N_ITEMS * (8 + 8) + 10 * 24, "scores f64 + ids + top-k entries"),
}
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "us": 1e-6,
         "nsecond": 1e-9, "ns": 1e-9, "msecond": 1e-3, "ms": 1e-3}


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, d = rows[0], rows[1], rows[2]
    return {m: (d[h.index(m)], u[h.index(m)]) for m in WANT if m in h}


def main(tag):
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = peaks["hbm_gbs"]
    lines = [f"# {tag}: ncu --set full of the C2 row kernels (one launch each)", "",
             "`tools/gpu_rowops_profiles.sh` (`ncu --set full --clock-control none -k regex:<k> -s 2 -c 1`"
             " on `bench.py --steps 1 --warmup 3`), summarised by `tools/ncu_rowops_summary.py`. "
             f"HBM peak = measured {hbm:.0f} GB/s (`MEASURED_PEAKS.json`). ncu times are cold-cache "
             "and serialised; DRAM bytes below the algorithmic bytes mean L2 absorbed part of the "
             "traffic (e.g. LN output still resident when the next GEMM reads it).", "",
             "| kernel | grid x block | regs | duration us | DRAM read MB | DRAM write MB | "
             "algorithmic MB | alg. GB/s | frac of HBM | ncu dram % | what |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for k, (alg, what) in ALG.items():
        p = os.path.join(ROOT, "gpurun_out", f"prof_{k}.ncu-rep")
        if not os.path.exists(p):
            continue
        r = raw(p)
        f = lambda m: float(r[m][0].replace(",", "")) * SCALE.get(r[m][1], 1)
        t = f("gpu__time_duration.sum")
        gbs = alg / t / 1e9
        lines.append(f"| `{k}` | {r['launch__grid_size'][0]} x {r['launch__block_size'][0]} | "
                     f"{r['launch__registers_per_thread'][0]} | {t * 1e6:.1f} | "
                     f"{f('dram__bytes_read.sum') / 1e6:.1f} | {f('dram__bytes_write.sum') / 1e6:.1f} | "
                     f"{alg / 1e6:.1f} | {gbs:.0f} | {gbs / hbm:.2f} | "
                     f"{float(r['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'][0]):.1f} | {what} |")
    lines += ["", "Reading: LayerNorm and embed+LN1 are HBM-bound streams; the score head "
              "(256 last rows) and the top-k (256 scores) are latency-bound launches (grid of "
              "32 / 1 CTAs): their bytes are ~1 MB, so their fraction of HBM is not the "
              "figure of merit — their ~15 us each is, against the 8.9 ms step."]
    out = os.path.join(ROOT, "profiles", f"{tag}_ncu_rowops.md")
    open(out, "w").write("\n".join(lines) + "\n")
    print(open(out).read())


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
