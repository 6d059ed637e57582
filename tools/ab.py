"""A/B device timing of library variants on the same box, interleaved.

    python tools/ab.py WORKLOAD LIB_A LIB_B [...]   (WORKLOAD: batch | ntt | ntt_batch | gcd | div | mul)

Each variant runs in its own process (MMM_CU_LIB=lib) `rounds` times,
alternating, and prints per-kernel-call CUDA-event times (min over reps).
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ["AB_ROOT"])
import paper_1402_0264_b200 as mmm
P = 469762049
w = os.environ["AB_WORK"]
rng = np.random.default_rng(7)
def draw(rows, terms):
    x = rng.integers(0, P, size=(rows, terms), dtype=np.int64).astype(np.uint32)
    x[:, -1] = rng.integers(1, P, size=rows, dtype=np.int64)
    return torch.from_numpy(x.view(np.int32)).cuda()
st = torch.cuda.current_stream().cuda_stream
calls = {}
if w == "batch":
    n, k = 4096, 4096
    A, B, Cd, D = draw(k, n), draw(k, n), draw(k, 2 * n), draw(k, n)
    F = torch.empty((k, 2 * n - 1), dtype=torch.int32, device="cuda")
    Q = torch.empty((k, n + 1), dtype=torch.int32, device="cuda")
    R = torch.empty((k, n - 1), dtype=torch.int32, device="cuda")
    calls["mul"] = lambda: mmm.mul_batched_dev(P, A.data_ptr(), n, n, B.data_ptr(), n, n, k, F.data_ptr(), 2 * n - 1, stream=st)
    calls["div"] = lambda: mmm.divmod_batched_dev(P, Cd.data_ptr(), 2 * n, 2 * n, D.data_ptr(), n, n, k, Q.data_ptr(), n + 1, R.data_ptr(), n - 1, stream=st)
elif w in ("ntt", "ntt_batch"):
    n, k = (1 << 20, 1) if w == "ntt" else (1 << 15, 256)  # cfg4: 2^21 product; 256 x 2^16 transforms
    A, B = draw(k, n), draw(k, n)
    F = torch.empty((k, 2 * n - 1), dtype=torch.int32, device="cuda")
    if k == 1:
        calls["ntt"] = lambda: mmm.ntt_mul_dev(P, A.data_ptr(), n, B.data_ptr(), n, F.data_ptr(), stream=st)
    else:
        calls["ntt"] = lambda: mmm.ntt_mul_batched_dev(P, A.data_ptr(), n, n, B.data_ptr(), n, n, k, F.data_ptr(), 2 * n - 1, stream=st)
elif w == "gcd":
    import bench
    g = bench.WORKLOADS["gcd"](0, bench.OursGen(42)); g.attach(mmm); g.device_setup()
    calls["gcd"] = lambda: g.device_step(st)
elif w == "div":
    A, B = draw(1, 1 << 16 | 1), draw(1, 1 << 15 | 1)
    Q = torch.empty(1 << 16, dtype=torch.int32, device="cuda"); R = torch.empty(1 << 16, dtype=torch.int32, device="cuda")
    s = int(os.environ.get("AB_S", "128"))
    calls["div"] = lambda: mmm.divmod_dev(P, A.data_ptr(), A.numel(), B.data_ptr(), B.numel(), Q.data_ptr(), R.data_ptr(), s=s, stream=st)
elif w == "mul":
    A, B = draw(1, 1 << 14), draw(1, 1 << 14)
    F = torch.empty(1 << 15, dtype=torch.int32, device="cuda")
    calls["mul"] = lambda: mmm.mul_dev(P, A.data_ptr(), A.numel(), B.data_ptr(), B.numel(), F.data_ptr(), s=int(os.environ.get("AB_S", "0")), stream=st)
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
reps = int(os.environ.get("AB_REPS", "10"))
out = []
for name, fn in calls.items():
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    out.append(f"{name} min {ts[0]*1e3:9.1f} us  med {ts[len(ts)//2]*1e3:9.1f} us")
print("  ".join(out), flush=True)
'''


def main():
    work, libs = sys.argv[1], sys.argv[2:]
    rounds = int(os.environ.get("AB_ROUNDS", "2"))
    for r in range(rounds):
        for lib in libs:
            env = dict(os.environ, MMM_CU_LIB=os.path.abspath(lib), AB_ROOT=ROOT, AB_WORK=work)
            res = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True,
                                 text=True, timeout=600)
            line = res.stdout.strip() or res.stderr.strip()[-400:]
            print(f"[{r}] {os.path.basename(os.path.dirname(lib)) or lib:>12s}: {line}", flush=True)


if __name__ == "__main__":
    main()
