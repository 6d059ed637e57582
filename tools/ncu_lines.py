#!/usr/bin/env python3
"""Map an ncu source-page CSV (SASS addresses) to CUDA source lines via the
cubin's line info: stall samples and excessive shared wavefronts per line.
    python tools/ncu_lines.py <src.csv> <object.o> <mangled-kernel-substring> [top]"""
import csv
import os
import re
import subprocess
import sys
import tempfile

src, obj, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 20
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
                   capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cub)],
                         capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(txt) if l.startswith("\t.section") and ".text." in l and kname in l)
off2line, cur = {}, None
for l in txt[start + 1:]:
    if l.startswith("\t.section") and ".text." in l:
        break
    if "//## File" in l:
        m, f = re.search(r"line (\d+)", l), re.search(r'File "([^"]+)"', l)
        if m:
            cur = (f.group(1).split("/")[-1] if f else "?", int(m.group(1)))
    mo = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if mo and cur:
        off2line[int(mo.group(1), 16)] = cur
rows = list(csv.reader(open(src)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
base = min(int(r[idx["Address"]], 16) for r in data)
S, X = "Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared Excessive"
REASONS = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg, exc, why = {}, {}, {}
for r in data:
    k = off2line.get(int(r[idx["Address"]], 16) - base, ("?", 0))
    agg[k] = agg.get(k, 0) + float(r[idx[S]] or 0)
    exc[k] = exc.get(k, 0) + float(r[idx[X]] or 0)
    w = why.setdefault(k, {})
    for h in REASONS:
        w[h] = w.get(h, 0) + float(r[idx[h]] or 0)
tot = sum(agg.values())
print(f"stall samples {tot:.0f}")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    rs = sorted(why[k].items(), key=lambda x: -x[1])[:3]
    rtxt = " ".join(f"{h[6:]}={100 * c / max(v, 1):.0f}%" for h, c in rs if c)
    print(f"  {k[0]}:{k[1]:5d}  {v:8.0f}  {100 * v / tot:5.1f}%  {rtxt}")
print("excessive shared wavefronts")
for k, v in sorted(exc.items(), key=lambda x: -x[1])[:10]:
    if v:
        print(f"  {k[0]}:{k[1]:5d}  {v:12.0f}")
