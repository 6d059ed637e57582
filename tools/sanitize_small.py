#!/usr/bin/env python3
"""Small cases of every entry point, for compute-sanitizer (memcheck):
    compute-sanitizer --tool memcheck python tools/sanitize_small.py
Each result is checked against the CPU oracle (C restatement)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1402_0264_b200 as mmm  # noqa: E402
from oracle import pyoracle  # noqa: E402

P = 469762049
port = pyoracle.Port()
rng = np.random.default_rng(5)


def r(p, n):
    x = rng.integers(0, p, n)
    x[-1] = max(int(x[-1]), 1)
    return x


for p in (P, 7, 2, 2147483647):
    for na, nb in ((1, 1), (33, 7), (300, 129), (1000, 999), (5000, 40)):
        a, b = r(p, na), r(p, nb)
        assert np.array_equal(mmm.mul(a, b, p, s=4), port.mul(a, b, p))
        q, rr = mmm.divmod(a, b, p, s=16)
        wq, wr = port.divmod(a, b, p)
        assert np.array_equal(q, wq) and np.array_equal(rr, wr)
        assert np.array_equal(mmm.gcd(a, b, p, s=8), port.gcd(a, b, p))
a, b = r(P, 20000), r(P, 9000)
for s in (1, 64, 128):
    q, rr = mmm.divmod(a, b, P, s=s)
    wq, wr = port.divmod(a, b, P)
    assert np.array_equal(q, wq) and np.array_equal(rr, wr), s
assert np.array_equal(mmm.ntt_mul(a, b, P), port.mul(a, b, P))
q, rr = mmm.divmod_fast(a, b, P)
assert np.array_equal(q, wq)
# batched: CUDA-core and tensor-core kernels, pipelined host path
for tc in ("0", "1"):
    os.environ["MMM_MUL_TC"] = tc
    os.environ["MMM_DIV_TC"] = tc
    A, B = rng.integers(0, P, (5, 700)), rng.integers(1, P, (5, 300))
    F = mmm.mul_batched(A, B, P)
    Q, R = mmm.divmod_batched(A, B, P)
    for i in range(5):
        assert np.array_equal(np.trim_zeros(F[i].astype(np.int64), "b"), port.mul(A[i], B[i], P))
        wq, wr = port.divmod(A[i], B[i], P)
        assert np.array_equal(np.trim_zeros(Q[i].astype(np.int64), "b"), wq)
        assert np.array_equal(np.trim_zeros(R[i].astype(np.int64), "b"), wr)
F = mmm.ntt_mul_batched(A, B, P)
assert np.array_equal(mmm.mul_batched_multi(A, B, P, [0, 0]), mmm.mul_batched(A, B, P))
print("sanitize_small: all cases match the oracle")
