#!/usr/bin/env python3
"""Run one workload instance through the device C-ABI (for ncu/sanitizer).

    python tools/prof_one.py gcd|mul|div|ntt|ntt_batch|mul_batch|div_batch [--s S] [--reps N]

Inputs are the bench's seed-42 configs; results are checked against the
golden digests so a profiled run is also a correct run."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--s", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    import paper_1402_0264_b200 as mmm
    mmm.load()
    w = bench.WORKLOADS[args.workload](args.s, bench.OursGen(42))
    w.attach(mmm)
    if getattr(w, "sharded", False):
        w.bind(bench.Dist("ours"))
    w.device_setup()
    sp = torch.cuda.current_stream().cuda_stream
    for _ in range(args.reps):
        w.device_step(sp)
    torch.cuda.synchronize()
    w.device_check()
    print(f"{args.workload}: ok, {mmm.launch_count()} launches")


if __name__ == "__main__":
    main()
