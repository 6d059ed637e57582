#!/usr/bin/env python3
"""Fold a round's ncu outputs into tracked profiles/ files.

    python tools/r2_merge.py gpurun_out/r2e r2e

* profiles/traffic.json -- DRAM bytes (read + write) per launch of each
  workload's kernels, from that workload's own `ncu --set full` capture (the
  `traffic` field bench.py reports; keyed by bench workload and kernel).
* profiles/<tag>_kernels.csv -- key metrics of every captured kernel.
* profiles/r2_s_sweep.csv -- the s sweep (tools/s_sweep.py: CUDA-event time
  and the paper's closed forms in ReportRow column order) with, per s, the
  blocked kernel's ncu counters: issued instructions, multiply-pipe (fmaheavy:
  IMAD/IMAD.WIDE/IMAD.HI) instructions and busy %, issue-active %, DRAM bytes
  and GB/s, L2 bytes.
"""
import csv
import json
import os
import re
import shutil
import sys

src, tag = sys.argv[1], sys.argv[2]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
CAPTURES = {"full_tcmul": "batch", "full_tcdiv": "batch", "full_gcd": "gcd", "full_mul": "mul",
            "full_div": "div", "full_ntt": "ntt", "full_ntt_batch": "ntt_batch"}


def short(kname):
    k = kname.replace("unnamed>::", "")
    m = re.search(r"(\w+)\s*[<(]", k.split("void ")[-1])
    return m.group(1) if m else k


def main():
    rows = list(csv.DictReader(open(os.path.join(src, "sum_kernels.csv"))))
    shutil.copy(os.path.join(src, "sum_kernels.csv"), os.path.join(PROF, f"{tag}_kernels.csv"))
    traffic_path = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    acc = {}
    for r in rows:
        cap = r["report"].replace(".ncu-rep", "")
        if cap not in CAPTURES or r["metric"] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        key = (CAPTURES[cap], short(r["kernel"]), cap)
        acc.setdefault(key, {"n": {}, "bytes": 0.0})
        v = float(r["value"]) * SCALE.get(r["unit"], 1)
        acc[key]["bytes"] += v
        acc[key]["n"][r["metric"]] = acc[key]["n"].get(r["metric"], 0) + 1
    for (w, k, cap), a in acc.items():
        launches = max(a["n"].values())
        traffic.setdefault(w, {})[k] = {
            "dram_bytes_per_launch": a["bytes"] / launches, "launches_captured": launches,
            "capture": f"{tag}:{cap}.ncu-rep (ncu --set full, tools/round2_ncu.sh)"}
    json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
    for f in os.listdir(src):
        if f.endswith("_brief.txt"):
            shutil.copy(os.path.join(src, f), os.path.join(PROF, f"{tag}_{f}"))
    # s sweep + per-s counters (rounds that re-ran it)
    if not os.path.exists(os.path.join(src, "s_sweep.csv")):
        print("traffic:", json.dumps(traffic, indent=1)[:1500])
        return
    sweep = list(csv.DictReader(open(os.path.join(src, "s_sweep.csv"))))
    cols = ["ncu_time_us", "inst_issued", "fmaheavy_inst", "fmaheavy_busy_pct", "issue_active_pct",
            "dram_read_B", "dram_write_B", "dram_GBps", "l2_bytes"]
    mm = {"gpu__time_duration.sum": "ncu_time_us", "sm__inst_issued.sum": "inst_issued",
          "sm__inst_executed_pipe_fmaheavy.sum": "fmaheavy_inst",
          "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active": "fmaheavy_busy_pct",
          "sm__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
          "dram__bytes_read.sum": "dram_read_B", "dram__bytes_write.sum": "dram_write_B",
          "dram__bytes.sum.per_second": "dram_GBps", "lts__t_bytes.sum": "l2_bytes"}
    for r in sweep:
        app = {"division": "div", "gcd": "gcd"}.get(r.get("algorithm") or r.get("app", ""))
        s = r.get("s")
        path = os.path.join(src, f"sweep_{app}_s{s}.csv") if app else None
        vals = {}
        if path and os.path.exists(path):
            lines = [ln for ln in open(path) if ln.startswith('"')]
            for q in csv.DictReader(lines):
                name, unit, v = q["Metric Name"], q["Metric Unit"], float(q["Metric Value"].replace(",", ""))
                if name not in mm:
                    continue
                if unit == "ns":
                    v /= 1e3
                elif unit == "byte/s":
                    v /= 1e9
                elif unit in SCALE:
                    v *= SCALE[unit]
                vals[mm[name]] = vals.get(mm[name], 0) + v  # summed over the call's kernels
            vals["kernel"] = ";".join(sorted({q["Kernel Name"].split("(")[0] for q in csv.DictReader(lines)}))
        for c in cols:
            r[c] = f"{vals[c]:.6g}" if c in vals else ""
        r["ncu_kernel"] = vals.get("kernel", "")
    out = os.path.join(PROF, "r2_s_sweep.csv")
    with open(out, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=list(sweep[0].keys()))
        w.writeheader()
        w.writerows(sweep)
    print("traffic:", json.dumps(traffic, indent=1)[:1500])
    print("wrote", out)


if __name__ == "__main__":
    main()
