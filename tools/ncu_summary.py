#!/usr/bin/env python3
"""Summarise ncu outputs brought back in gpurun_out/ into profiles/ (tracked).

    python tools/ncu_summary.py gpurun_out/r1 profiles/r1

Writes <out>_launches.csv (kernel, launches, total us, share) from the
launch-list pass and <out>_kernels.csv (key metrics per --set full capture).
"""
import csv
import glob
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__average_warp_latency_issue_stalled_wait", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            k = r[hdr.index("Kernel Name")]
            v, u = float(r[hdr.index("Metric Value")]), r[hdr.index("Metric Unit")]
            us = v / 1e3 if u == "ns" else v * 1e3 if u == "ms" else v
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1
            a[1] += us
    tot = sum(v[1] for v in agg.values()) or 1.0
    with open(out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["kernel", "launches", "total_us", "share"])
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            w.writerow([k, n, f"{t:.1f}", f"{t / tot:.4f}"])


def kernels(reps, out):
    with open(out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["report", "kernel", "metric", "unit", "value"])
        for rep in reps:
            raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                 text=True).stdout
            r = list(csv.reader(raw.splitlines()))
            if len(r) < 3:
                continue
            h, units = r[0], r[1]
            for vals in r[2:]:  # every captured launch
                kname = vals[h.index("Kernel Name")] if "Kernel Name" in h else "?"
                for key in KEYS:
                    if key in h:
                        i = h.index(key)
                        w.writerow([os.path.basename(rep), kname, key, units[i], vals[i]])


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(os.path.dirname(dst) or ".", exist_ok=True)
    for f in glob.glob(os.path.join(src, "launches_*.csv")):
        tag = os.path.basename(f)[len("launches_"):-4]
        launches(f, f"{dst}_launches_{tag}.csv")
    reps = sorted(glob.glob(os.path.join(src, "*.ncu-rep")))
    if reps:
        kernels(reps, f"{dst}_kernels.csv")


if __name__ == "__main__":
    main()
