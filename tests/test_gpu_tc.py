"""GPU parity of the tensor-core batched product (csrc/tcmul.cu: tcgen05
kind::i8 limb-split Toeplitz GEMM) against the CPU oracle and the IMAD.WIDE
product kernel: bit-exact for every shape class it accepts (1..4096 terms per
operand, ragged block edges, odd/even Toeplitz offsets, primes from 2 to
2^31 - 1, limb values up to 255 in every position)."""
import numpy as np
import pytest

import suites

pytestmark = pytest.mark.gpu

P = suites.P_BENCH


def _batch(rng, p, cnt, na, nb, extreme=False):
    if extreme:  # every limb 255 where p allows: the s32 accumulation bound
        A = np.full((cnt, na), p - 1, dtype=np.int64)
        B = np.full((cnt, nb), p - 1, dtype=np.int64)
    else:
        A = rng.integers(0, p, (cnt, na))
        B = rng.integers(0, p, (cnt, nb))
    return A, B


@pytest.mark.parametrize("p", [P, 2147483647, 2013265921, 101, 7, 2])
def test_tc_product_vs_oracle(cuda_lib, port, monkeypatch, p):
    mmm = cuda_lib
    rng = np.random.default_rng(p % 10007)
    monkeypatch.setenv("MMM_MUL_TC", "1")
    shapes = [(1, 1), (1, 4096), (4096, 1), (128, 128), (129, 127), (1000, 3000), (4096, 4096),
              (4095, 4093), (257, 4096), (4096, 300)]
    for na, nb in shapes:
        A, B = _batch(rng, p, 3, na, nb)
        F = mmm.mul_batched(A, B, p)
        for i in range(3):
            want = port.mul(A[i], B[i], p)
            got = np.trim_zeros(F[i].astype(np.int64), "b")
            assert np.array_equal(got, want), (p, na, nb, i)


def test_tc_product_accumulation_bound(cuda_lib, port, monkeypatch):
    """All coefficients p - 1 (limbs 0xFF where possible): the largest plane sums."""
    mmm = cuda_lib
    monkeypatch.setenv("MMM_MUL_TC", "1")
    for p in (2147483647, P):
        A, B = _batch(None, p, 2, 4096, 4096, extreme=True)
        F = mmm.mul_batched(A, B, p)
        want = port.mul(A[0], B[0], p)
        assert np.array_equal(F[0].astype(np.int64), want)
        assert np.array_equal(F[1], F[0])


def test_tc_product_equals_imad_kernel_large_batch(cuda_lib, monkeypatch):
    """A batch larger than the grid (instances walk the persistent CTAs) with
    strided rows: tensor-core and IMAD.WIDE kernels agree word for word."""
    import torch
    mmm = cuda_lib
    rng = np.random.default_rng(3)
    cnt, na, nb = 400, 2048, 1500
    A = rng.integers(0, P, (cnt, na + 5)).astype(np.uint32)
    B = rng.integers(0, P, (cnt, nb + 3)).astype(np.uint32)
    dA = torch.from_numpy(A.view(np.int32)).cuda()
    dB = torch.from_numpy(B.view(np.int32)).cuda()
    nf = na + nb - 1
    outs = []
    for tc in ("1", "0"):
        monkeypatch.setenv("MMM_MUL_TC", tc)
        dF = torch.full((cnt, nf + 7), -1, dtype=torch.int32, device="cuda")
        mmm.mul_batched_dev(P, dA.data_ptr(), na + 5, na, dB.data_ptr(), nb + 3, nb, cnt,
                            dF.data_ptr(), nf + 7, stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        outs.append(dF.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    assert (outs[0][:, nf:] == -1).all()  # nothing written past each row


def test_tc_product_fanout(cuda_lib, monkeypatch):
    import torch
    mmm = cuda_lib
    monkeypatch.setenv("MMM_MUL_TC", "1")
    rng = np.random.default_rng(4)
    cnt, n = 5, 700
    A = rng.integers(0, P, (cnt, n)).astype(np.uint32)
    dA = torch.from_numpy(A.view(np.int32)).cuda()
    outs = [torch.zeros((cnt, 2 * n - 1), dtype=torch.int32, device="cuda") for _ in range(3)]
    mmm.mul_batched_fanout_dev(P, dA.data_ptr(), n, n, dA.data_ptr(), n, n, cnt,
                               [o.data_ptr() for o in outs], 2 * n - 1,
                               stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    want = mmm.mul_batched(A, A, P)
    for o in outs:
        assert np.array_equal(o.cpu().numpy().view(np.uint32), want)


# ------------------------------------------------ tensor-core division ----
@pytest.mark.parametrize("p", [P, 2147483647, 101, 7, 2])
def test_tc_division_vs_oracle(cuda_lib, port, monkeypatch, p):
    """csrc/tcdiv.cu (128 heads per step, remainder accumulated on the tensor
    core) == oracle_divmod, including quotient lengths that are not multiples
    of 128, mu = 1, 2-term divisors and degree drops over small fields."""
    mmm = cuda_lib
    monkeypatch.setenv("MMM_DIV_TC", "1")
    rng = np.random.default_rng(77 + p % 1000)
    shapes = [(8192, 4096), (8191, 4096), (5000, 3000), (4096, 4096), (4097, 4096), (8192, 2),
              (300, 129), (1000, 999), (8192, 129), (130, 2), (6000, 700), (257, 128)]
    for na, nb in shapes:
        A = rng.integers(0, p, (2, na))
        B = rng.integers(0, p, (2, nb))
        B[:, -1] = np.maximum(B[:, -1], 1)
        Q, R = mmm.divmod_batched(A, B, p)
        for i in range(2):
            wq, wr = port.divmod(A[i], B[i], p)
            assert np.array_equal(np.trim_zeros(Q[i].astype(np.int64), "b"), wq), (p, na, nb, i)
            assert np.array_equal(np.trim_zeros(R[i].astype(np.int64), "b"), wr), (p, na, nb, i)


def test_tc_division_equals_cta_kernel(cuda_lib, monkeypatch):
    """Many instances (the persistent grid walks the batch), strided rows:
    tensor-core and CUDA-core division agree word for word."""
    mmm = cuda_lib
    rng = np.random.default_rng(8)
    cnt, na, nb = 300, 8192, 4096
    A = rng.integers(0, P, (cnt, na))
    B = rng.integers(0, P, (cnt, nb))
    B[:, -1] = np.maximum(B[:, -1], 1)
    outs = []
    for tc in ("1", "0"):
        monkeypatch.setenv("MMM_DIV_TC", tc)
        outs.append(mmm.divmod_batched(A, B, P))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_tc_division_fanout(cuda_lib, port, monkeypatch):
    """The tensor-core division's fan-out epilogue (q and r into every pointer
    of a set, as the sharded cfg5 gather uses it)."""
    import torch
    mmm = cuda_lib
    monkeypatch.setenv("MMM_DIV_TC", "1")
    rng = np.random.default_rng(12)
    cnt, na, nb = 5, 3000, 1300
    A = rng.integers(0, P, (cnt, na)).astype(np.uint32)
    B = rng.integers(1, P, (cnt, nb)).astype(np.uint32)
    dA = torch.from_numpy(A.view(np.int32)).cuda()
    dB = torch.from_numpy(B.view(np.int32)).cuda()
    lq, lr = na - nb + 1, nb - 1
    qs = [torch.zeros((cnt, lq), dtype=torch.int32, device="cuda") for _ in range(3)]
    rs = [torch.zeros((cnt, lr), dtype=torch.int32, device="cuda") for _ in range(3)]
    mmm.divmod_batched_fanout_dev(P, dA.data_ptr(), na, na, dB.data_ptr(), nb, nb, cnt,
                                  [q.data_ptr() for q in qs], lq, [r.data_ptr() for r in rs], lr,
                                  stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for i in range(cnt):
        wq, wr = port.divmod(A[i], B[i], P)
        for q, r in zip(qs, rs):
            assert np.array_equal(np.trim_zeros(q[i].cpu().numpy().view(np.uint32).astype(np.int64), "b"), wq)
            assert np.array_equal(np.trim_zeros(r[i].cpu().numpy().view(np.uint32).astype(np.int64), "b"), wr)


# ------------------------------------------- one large product, split ----
@pytest.mark.parametrize("p", [P, 2147483647, 7])
def test_tc_single_product_vs_oracle(cuda_lib, port, monkeypatch, p):
    """csrc/tcmul.cu tcmul_split_kernel (segments of 4096 terms x tile ranges
    over the SMs, u64 accumulation, grid-wide finalise) == oracle_mul."""
    mmm = cuda_lib
    monkeypatch.setenv("MMM_MUL_TC", "1")
    rng = np.random.default_rng(31 + p % 97)
    for na, nb in [(1, 1), (5000, 3), (4096, 4096), (4097, 4095), (9000, 5000), (16384, 1000),
                   (700, 20000)]:
        a, b = rng.integers(0, p, na), rng.integers(0, p, nb)
        a[-1] = max(int(a[-1]), 1)
        b[-1] = max(int(b[-1]), 1)
        got = mmm.mul(a, b, p)
        want = port.mul(a, b, p) if na * nb <= 5e7 else mmm.ntt_mul(a, b, p) if p == P else None
        if want is None:
            monkeypatch.setenv("MMM_MUL_TC", "0")
            want = mmm.mul(a, b, p, s=8)
            monkeypatch.setenv("MMM_MUL_TC", "1")
        assert np.array_equal(got, want), (p, na, nb)
    # repeated calls reuse the zeroed accumulator
    a, b = rng.integers(0, p, 12000), rng.integers(0, p, 12000)
    assert np.array_equal(mmm.mul(a, b, p), mmm.mul(a, b, p))


def test_cfg1_tensor_core(cuda_lib, golden_configs):
    """cfg1 (2^14 x 2^14) on the default (auto) path == the reference digest."""
    from helpers import ProductRng, digest
    c = suites.cfg1(ProductRng(42))
    assert digest(cuda_lib.mul(c["a"], c["b"], P)) == golden_configs["cfg1"]["f"]
