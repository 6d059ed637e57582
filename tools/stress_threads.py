"""Concurrency stress of the host C ABI: several Python threads call divmod / mul on their own
per-thread streams (tests/test_gpu_coverage.py::test_scratch_across_streams_and_threads, in a loop).
    python tools/stress_threads.py [rounds] [mode: both|div|mul] [s] [release: 0|1]"""
import os, sys, threading
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1402_0264_b200 as mmm
from oracle import pyoracle

P = 469762049
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 20
mode = sys.argv[2] if len(sys.argv) > 2 else "both"
s = int(sys.argv[3]) if len(sys.argv) > 3 else 64
rel = int(sys.argv[4]) if len(sys.argv) > 4 else 1
port = pyoracle.Port()
rng = np.random.default_rng(31)
def rand(n):
    x = rng.integers(0, P, size=n, dtype=np.int64).astype(np.uint32)
    x[-1] = rng.integers(1, P)
    return x
cases = []
for _ in range(4):
    a, b = rand(20000), rand(9000)
    cases.append((a, b, port.divmod(a, b, P), port.mul(a[:3000], b[:2000], P)))
gcases = []
if mode == "gcd":
    for _ in range(2):
        gg, u, v = rand(1200), rand(2400), rand(2399)
        ga, gb = port.mul(gg, u, P), port.mul(gg, v, P)
        gcases.append((ga, gb, port.gcd(ga, gb, P)))
bad = []
def worker(k, rd):
    try:
        if mode == "gcd":  # two threads run GCDs, two run products and divisions beside them
            for i in range(3):
                if k < 2:
                    ga, gb, wg = gcases[(k + i) % 2]
                    got = mmm.gcd(ga, gb, P, s=s)
                    if not np.array_equal(got, wg):
                        bad.append(("gcd", rd, k, i, len(got), len(wg)))
                else:
                    a, b, (wq, wr), wm = cases[(k + i) % 4]
                    if not np.array_equal(mmm.mul(a[:3000], b[:2000], P), wm):
                        bad.append(("mul-beside-gcd", rd, k, i))
                    q, r = mmm.divmod(a, b, P, s=128)
                    if not (np.array_equal(q, wq) and np.array_equal(r, wr)):
                        bad.append(("div-beside-gcd", rd, k, i))
            return
        for i, (a, b, (wq, wr), wm) in enumerate(cases[k:] + cases[:k]):
            if mode in ("both", "div"):
                q, r = mmm.divmod(a, b, P, s=s)
                if not (np.array_equal(q, wq) and np.array_equal(r, wr)):
                    dq = np.nonzero(q != wq)[0] if len(q) == len(wq) else [-1]
                    dr = np.nonzero(r != wr)[0] if len(r) == len(wr) else [-1]
                    bad.append(("div", rd, k, i, len(dq), (int(dq[0]), int(dq[-1])) if len(dq) else None,
                                len(dr), (int(dr[0]), int(dr[-1])) if len(dr) else None))
            if mode in ("both", "mul"):
                m = mmm.mul(a[:3000], b[:2000], P)
                if not np.array_equal(m, wm):
                    dm = np.nonzero(m != wm)[0] if len(m) == len(wm) else [-1]
                    bad.append(("mul", rd, k, i, len(dm), (int(dm[0]), int(dm[-1]))))
        if rel:
            mmm.release_scratch()
    except Exception as e:  # noqa: BLE001
        bad.append(("exc", rd, k, repr(e)[:200]))
phase1 = int(sys.argv[5]) if len(sys.argv) > 5 else 0
def multi_stream():
    import torch
    streams = [torch.cuda.Stream() for _ in range(3)]
    outs = []
    for i, (a, b, _, _) in enumerate(cases * 2):
        st = streams[i % 3]
        with torch.cuda.stream(st):
            da = torch.from_numpy(a.astype(np.uint32).view(np.int32)).cuda()
            db = torch.from_numpy(b.astype(np.uint32).view(np.int32)).cuda()
            dq = torch.zeros(len(a) - len(b) + 1, dtype=torch.int32, device="cuda")
            dr = torch.zeros(len(b) - 1, dtype=torch.int32, device="cuda")
            mmm.divmod_dev(P, da.data_ptr(), len(a), db.data_ptr(), len(b), dq.data_ptr(),
                           dr.data_ptr(), s=128, stream=st.cuda_stream)
            outs.append((dq, dr))
    torch.cuda.synchronize()
    for i, ((dq, dr), (_, _, (wq, wr), _)) in enumerate(zip(outs, cases * 2)):
        q = np.trim_zeros(dq.cpu().numpy().view(np.uint32), "b")
        r = np.trim_zeros(dr.cpu().numpy().view(np.uint32), "b")
        if not (np.array_equal(q, wq) and np.array_equal(r, wr)):
            bad.append(("phase1", i))
for rd in range(rounds):
    if phase1:
        multi_stream()
    ts = [threading.Thread(target=worker, args=(k, rd)) for k in range(4)]
    for t in ts: t.start()
    for t in ts: t.join()
print(f"mode={mode} s={s} release={rel} rounds={rounds}: {len(bad)} bad")
for b in bad[:12]: print("  ", b)
