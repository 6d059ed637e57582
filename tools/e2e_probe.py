"""cfg5 end-to-end anatomy: PCIe rates, each batched host call timed alone
(wall clock around the synchronous C-ABI call, pinned inputs and results),
the device-only kernels, and (MMM_TC_STATS=1) tcdiv's phase clocks.

    python tools/e2e_probe.py [reps]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1402_0264_b200 as mmm  # noqa: E402

P = 469762049
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5


def pinned(x):
    t = torch.from_numpy(np.ascontiguousarray(x).view(np.int32)).pin_memory()
    return t.numpy().view(np.uint32), t


def bw():
    n = 335 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"pcie {name}: {n / e0.elapsed_time(e1) / 1e6:.1f} GB/s", flush=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    print(f"pcie both directions: {2 * n / (time.perf_counter() - t0) / 1e9:.1f} GB/s total",
          flush=True)


def timeit(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts), float(np.median(ts))


def main():
    torch.cuda.init()
    bw()
    rng = np.random.default_rng(42)  # timing only: any canonical inputs, nonzero leads
    def draw(rows, terms):
        x = rng.integers(0, P, size=(rows, terms), dtype=np.int64).astype(np.uint32)
        x[:, -1] = rng.integers(1, P, size=rows, dtype=np.int64)
        return pinned(x)[0]
    A, B, Cd, D = draw(4096, 4096), draw(4096, 4096), draw(4096, 8192), draw(4096, 4096)
    n = A.shape[1]
    k = A.shape[0]
    hF = pinned(np.zeros((k, 2 * n - 1), np.uint32))[0]
    hQ = pinned(np.zeros((k, n + 1), np.uint32))[0]
    hR = pinned(np.zeros((k, n - 1), np.uint32))[0]
    m = timeit(lambda: mmm.mul_batched(A, B, P, out=hF), reps)
    print(f"mul_batched e2e: min {m[0]:.3f} ms median {m[1]:.3f} ms", flush=True)
    d = timeit(lambda: mmm.divmod_batched(Cd, D, P, q_out=hQ, r_out=hR), reps)
    print(f"divmod_batched e2e: min {d[0]:.3f} ms median {d[1]:.3f} ms", flush=True)
    dA, dB, dC, dD = (torch.from_numpy(x.view(np.int32)).cuda() for x in (A, B, Cd, D))
    dF = torch.empty((k, 2 * n - 1), dtype=torch.int32, device="cuda")
    dQ = torch.empty((k, n + 1), dtype=torch.int32, device="cuda")
    dR = torch.empty((k, n - 1), dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def dev_mul():
        mmm.mul_batched_dev(P, dA.data_ptr(), n, n, dB.data_ptr(), n, n, k, dF.data_ptr(),
                            2 * n - 1, stream=st)
        torch.cuda.synchronize()

    def dev_div():
        mmm.divmod_batched_dev(P, dC.data_ptr(), 2 * n, 2 * n, dD.data_ptr(), n, n, k,
                               dQ.data_ptr(), n + 1, dR.data_ptr(), n - 1, stream=st)
        torch.cuda.synchronize()

    m = timeit(dev_mul, reps)
    print(f"mul_batched_dev: min {m[0]:.3f} ms", flush=True)
    d = timeit(dev_div, reps)
    print(f"divmod_batched_dev: min {d[0]:.3f} ms", flush=True)
    for kk in (512, 1024, 2048):
        def dev_div_k(kk=kk):
            mmm.divmod_batched_dev(P, dC.data_ptr(), 2 * n, 2 * n, dD.data_ptr(), n, n, kk,
                                   dQ.data_ptr(), n + 1, dR.data_ptr(), n - 1, stream=st)
            torch.cuda.synchronize()
        d = timeit(dev_div_k, reps)
        print(f"divmod_batched_dev count={kk}: min {d[0]:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
