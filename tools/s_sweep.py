#!/usr/bin/env python3
"""Model-vs-measured blocking sweep.

    python tools/s_sweep.py [--out profiles/r1_s_sweep.csv] [--reps 5]

For the three blocked programs on their BASELINE configs -- cfg3 division
(s heads per grid step), cfg2 GCD (s eliminations per matrix batch, capped by
the 64-word matrix), cfg1 multiplication (s x s register tiles) -- times the
B200 kernel at each s (CUDA events on the launch stream, median of --reps,
result checked against the golden digest) and prints the paper's closed forms
(paper_1402_0264_b200.costmodel, a restatement of proj/src/costmodel.cpp) for
the same (n, m, s): predicted W, S, O, N, L, C and the Graham-Brent estimate
(N/P + L)*C with P = the SM count.  Output: ReportRow columns in the
reference's order, then gpu_ms, gpu_rel (time / best time of the sweep),
model_rel (T_bound / best T_bound of the sweep) and grid_steps.
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1402_0264_b200 import costmodel as cm  # noqa: E402

U = 2  # the model's word-transfer cost default (costmodel.hpp CostInputs::U)


def time_ms(w, reps):
    import torch
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w.device_step(st.cuda_stream)  # warm (allocator, first launch)
    st.synchronize()
    w.device_check()
    out = []
    for _ in range(reps):
        e0.record(st)
        w.device_step(st.cuda_stream)
        e1.record(st)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_s_sweep.csv"))
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    P = torch.cuda.get_device_properties(0).multi_processor_count
    rows = []

    def sweep(app, variant, name, svals, model, steps):
        got = []
        for s in svals:
            import paper_1402_0264_b200 as mmm
            w = bench.WORKLOADS[name](s, bench.OursGen(42))
            w.attach(mmm)
            w.device_setup()
            ms = time_ms(w, args.reps)
            n, m, t = model(w, s)
            tb = cm.graham_brent_bound(t.N, t.L, t.C, P)
            r = cm.row(app, variant, n=n, m=m, l=t_l(app), s=s, U=U, pred=t, T_bound=tb,
                       meas={"L": steps(w, s)} if steps(w, s) is not None else None)
            r["gpu_ms"], r["grid_steps"] = f"{ms:.4f}", steps(w, s)
            got.append((r, ms, tb))
            print(f"{app:15s} s={s:4d}  {ms:9.3f} ms  model T={float(tb):.4g}", flush=True)
        best_ms = min(g[1] for g in got)
        best_tb = min(g[2] for g in got)
        for r, ms, tb in got:
            r["gpu_rel"] = f"{ms / best_ms:.4f}"
            r["model_rel"] = f"{float(tb / best_tb):.4f}"
            rows.append(r)

    def t_l(app):
        return 128 if app == "multiplication" else None

    # cfg3 division: n = 2^16+1, m = 2^15+1 terms; one grid step per s heads
    mu = (1 << 16) - (1 << 15) + 1
    sweep("division", cm.OPTIMIZED, "div", [1, 2, 4, 8, 16, 32, 64, 128, 256, 512],
          lambda w, s: ((1 << 16) + 1, (1 << 15) + 1,
                        cm.division_cost(cm.OPTIMIZED, (1 << 16) + 1, (1 << 15) + 1, s=s, U=U)),
          lambda w, s: -(-mu // s))
    # cfg2 gcd: n = 12289, m = 12288 terms; batches of <= s eliminations (matrix cap 64)
    sweep("gcd", cm.OPTIMIZED, "gcd", [2, 4, 8, 16, 32, 64, 128],
          lambda w, s: (len(w.a), len(w.b), cm.gcd_cost(cm.OPTIMIZED, len(w.a), len(w.b), s=s, U=U)),
          lambda w, s: None)
    # cfg1 multiplication: n = m = 2^14; s x s tiles, l = 128 threads per block
    sweep("multiplication", "", "mul", [1, 2, 4, 8, 16],
          lambda w, s: (1 << 14, 1 << 14, cm.multiplication_cost(1 << 14, 1 << 14, l=128, s=s, U=U)),
          lambda w, s: 1)
    text = cm.to_csv(rows, extra=("gpu_ms", "gpu_rel", "model_rel", "grid_steps"))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        fh.write(text)
    print(f"wrote {args.out} ({len(rows)} rows, P = {P})")


if __name__ == "__main__":
    main()
