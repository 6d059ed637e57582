"""GPU parity for the shapes round 1 left open, the several-GPU C ABI, and the
host-path plumbing (per-thread scratch, caller-supplied outputs).

* Division by short divisors (1..16 terms) of long dividends (>= 10^5 terms),
  single and batched, every schedule: exactly oracle_divmod
  (/root/reference/proj/src/oracle.cpp:51-67).
* Config-scale GCD (cfg2 shapes) over GF(2), GF(7), GF(101) and GF(2^31-1),
  where degree drops are frequent: exactly oracle_gcd
  (oracle.cpp:69-78), checked against the CPU oracle at full size.
* cfg3-shape division at p = 2^31 - 1.
* mmm_cu_*_batched_multi(_dev): shares over a device list (repeats allowed,
  so the scatter / fused-gather path runs on one GPU) == the single call.
"""
import threading

import numpy as np
import pytest

from helpers import PortRng
import suites

pytestmark = pytest.mark.gpu

P = suites.P_BENCH
P31 = 2147483647


def _rand(rng, p, n):
    x = rng.integers(0, p, n)
    x[-1] = max(int(x[-1]), 1)
    return x


# ------------------------------------------------ short divisors, long a --
@pytest.mark.parametrize("p", [P, P31, 7, 2])
def test_division_short_divisors_long_dividends(cuda_lib, port, p):
    mmm = cuda_lib
    rng = np.random.default_rng(1000 + p % 997)
    for na in (100_001, 150_000):
        a = _rand(rng, p, na)
        for nb in (1, 2, 3, 5, 8, 16):
            b = _rand(rng, p, nb)
            wq, wr = port.divmod(a, b, p)
            for s in (1, 8, 64, 128):
                q, r = mmm.divmod(a, b, p, s=s)
                assert np.array_equal(q, wq) and np.array_equal(r, wr), (p, na, nb, s)


@pytest.mark.parametrize("sched", ["grid", "pipe"])
def test_division_forced_schedules_short_divisors(cuda_lib, port, sched, monkeypatch):
    """Both single-instance schedules at divisor lengths below their usual
    range (the dispatcher sends these to the grid; forcing covers the rest)."""
    monkeypatch.setenv("MMM_DIV_SCHED", sched)
    rng = np.random.default_rng(4)
    for na, nb in [(60_000, 2), (60_000, 17), (30_001, 300), (40_000, 1100)]:
        a, b = _rand(rng, P, na), _rand(rng, P, nb)
        wq, wr = port.divmod(a, b, P)
        for s in (32, 128):
            q, r = cuda_lib.divmod(a, b, P, s=s)
            assert np.array_equal(q, wq) and np.array_equal(r, wr), (sched, na, nb, s)


def test_division_by_constant_batched(cuda_lib, port):
    mmm = cuda_lib
    rng = np.random.default_rng(8)
    for p in (P, P31, 2):
        for na in (1, 7, 5000, 120_000):
            A = rng.integers(0, p, (3, na))
            B = rng.integers(1, p, (3, 1))
            Q, R = mmm.divmod_batched(A, B, p, s=16)
            assert R.shape == (3, 0)
            for i in range(3):
                wq, wr = port.divmod(A[i], B[i], p)
                assert np.array_equal(np.trim_zeros(Q[i], "b"), wq) and wr.size == 0, (p, na, i)


def test_division_batched_instances_beyond_one_cta(cuda_lib, port):
    """Batched instances whose dividend does not fit one CTA's shared memory run
    one single-instance division each (the row results are then copied out)."""
    mmm = cuda_lib
    rng = np.random.default_rng(9)
    for na, nb in [(60_000, 3000), (70_000, 5)]:
        A = rng.integers(0, P, (3, na))
        B = rng.integers(0, P, (3, nb))
        B[:, -1] = np.maximum(B[:, -1], 1)
        Q, R = mmm.divmod_batched(A, B, P, s=64)
        for i in range(3):
            wq, wr = port.divmod(A[i], B[i], P)
            assert np.array_equal(np.trim_zeros(Q[i], "b"), wq)
            assert np.array_equal(np.trim_zeros(R[i], "b"), wr)


# ------------------------------------------------ config-scale GCD, p --
@pytest.mark.parametrize("p", [2, 7, 101, P31])
def test_cfg2_shape_gcd_other_primes(cuda_lib, port, p):
    """cfg2's shapes (deg g = 2^12, deg u = 2^13, deg v = 2^13 - 1) with the
    same draw order as BASELINE configs[1], over other primes."""
    rng = PortRng(port, 42)
    g = port.monic(rng.random_poly((1 << 12) + 1, p), p)
    u = rng.random_poly((1 << 13) + 1, p)
    v = rng.random_poly(1 << 13, p)
    a, b = port.mul(g, u, p), port.mul(g, v, p)
    want = port.gcd(a, b, p)
    assert len(want) >= len(g)
    for s in (8, 64, 128):
        assert np.array_equal(cuda_lib.gcd(a, b, p, s=s), want), (p, s)


def test_cfg3_shape_division_p31(cuda_lib, port):
    rng = PortRng(port, 42)
    a = rng.random_poly((1 << 16) + 1, P31)
    b = rng.random_poly((1 << 15) + 1, P31)
    wq, wr = port.divmod(a, b, P31)
    for s in (8, 128):
        q, r = cuda_lib.divmod(a, b, P31, s=s)
        assert np.array_equal(q, wq) and np.array_equal(r, wr), s
    q, r = cuda_lib.divmod_fast(a, b, P31)
    assert np.array_equal(q, wq) and np.array_equal(r, wr)


# ---------------------------------------------------- several devices --
DEVICE_LISTS = [[0], [0, 0], [0, 0, 0]]


@pytest.mark.parametrize("devs", DEVICE_LISTS)
def test_multi_host_batches(cuda_lib, devs):
    mmm = cuda_lib
    rng = np.random.default_rng(21)
    A, B = rng.integers(0, P, (7, 500)), rng.integers(0, P, (7, 300))
    B[:, -1] = np.maximum(B[:, -1], 1)
    assert np.array_equal(mmm.mul_batched_multi(A, B, P, devs), mmm.mul_batched(A, B, P))
    q1, r1 = mmm.divmod_batched_multi(A, B, P, devs)
    q0, r0 = mmm.divmod_batched(A, B, P)
    assert np.array_equal(q1, q0) and np.array_equal(r1, r0)
    assert np.array_equal(mmm.ntt_mul_batched_multi(A, B, P, devs),
                          mmm.ntt_mul_batched(A, B, P))
    # fewer instances than devices: empty shares
    assert np.array_equal(mmm.mul_batched_multi(A[:2], B[:2], P, devs),
                          mmm.mul_batched(A[:2], B[:2], P))


def test_multi_host_errors(cuda_lib):
    mmm = cuda_lib
    A = np.ones((4, 8), dtype=np.uint32)
    with pytest.raises(mmm.InvalidArgument):
        mmm.mul_batched_multi(A, A, P, [0, 999])
    with pytest.raises(mmm.InvalidArgument):
        mmm.mul_batched_multi(A, A, P, [])
    bad = A.copy()
    bad[3, 2] = P  # non-canonical coefficient in the last share
    with pytest.raises(mmm.InvalidArgument, match="share"):
        mmm.mul_batched_multi(bad, A, P, [0, 0])


@pytest.mark.parametrize("devs", DEVICE_LISTS)
def test_multi_dev_batches(cuda_lib, devs):
    import torch
    mmm = cuda_lib
    rng = np.random.default_rng(22)
    cnt, na, nb = 9, 700, 400
    A, B = rng.integers(0, P, (cnt, na)), rng.integers(0, P, (cnt, nb))
    B[:, -1] = np.maximum(B[:, -1], 1)
    dA = torch.from_numpy(A.astype(np.uint32).view(np.int32)).cuda()
    dB = torch.from_numpy(B.astype(np.uint32).view(np.int32)).cuda()
    st = torch.cuda.current_stream().cuda_stream
    nf = na + nb - 1
    dF = torch.full((cnt, nf + 3), -1, dtype=torch.int32, device="cuda")  # ldf > nf
    mmm.mul_batched_multi_dev(P, dA.data_ptr(), na, na, dB.data_ptr(), nb, nb, cnt,
                              dF.data_ptr(), nf + 3, devs, stream=st)
    want = mmm.mul_batched(A, B, P)
    assert np.array_equal(dF[:, :nf].cpu().numpy().view(np.uint32), want)
    dQ = torch.zeros((cnt, na - nb + 1), dtype=torch.int32, device="cuda")
    dR = torch.zeros((cnt, nb - 1), dtype=torch.int32, device="cuda")
    mmm.divmod_batched_multi_dev(P, dA.data_ptr(), na, na, dB.data_ptr(), nb, nb, cnt,
                                 dQ.data_ptr(), na - nb + 1, dR.data_ptr(), nb - 1, devs,
                                 stream=st)
    q0, r0 = mmm.divmod_batched(A, B, P)
    assert np.array_equal(dQ.cpu().numpy().view(np.uint32), q0)
    assert np.array_equal(dR.cpu().numpy().view(np.uint32), r0)
    for ldf in (nf, nf + 3):
        dF.fill_(-1)
        mmm.ntt_mul_batched_multi_dev(P, dA.data_ptr(), na, na, dB.data_ptr(), nb, nb, cnt,
                                      dF.data_ptr(), ldf, devs, stream=st)
        got = dF.view(-1)[: cnt * ldf].view(cnt, ldf)[:, :nf].cpu().numpy().view(np.uint32)
        assert np.array_equal(got, want), ldf


# ------------------------------------------------ host-path plumbing --
def test_scratch_across_streams_and_threads(cuda_lib, port):
    """Per-thread arenas: calls alternating between streams (reuse ordered by
    the arena's event), calls from short-lived threads, release in between."""
    import torch
    mmm = cuda_lib
    rng = np.random.default_rng(31)
    cases = []
    for _ in range(4):
        a, b = _rand(rng, P, 20000), _rand(rng, P, 9000)
        cases.append((a, b, port.divmod(a, b, P)))
    streams = [torch.cuda.Stream() for _ in range(3)]
    outs = []
    for i, (a, b, _) in enumerate(cases * 2):
        s = streams[i % 3]
        with torch.cuda.stream(s):
            da = torch.from_numpy(a.astype(np.uint32).view(np.int32)).cuda()
            db = torch.from_numpy(b.astype(np.uint32).view(np.int32)).cuda()
            dq = torch.zeros(len(a) - len(b) + 1, dtype=torch.int32, device="cuda")
            dr = torch.zeros(len(b) - 1, dtype=torch.int32, device="cuda")
            mmm.divmod_dev(P, da.data_ptr(), len(a), db.data_ptr(), len(b), dq.data_ptr(),
                           dr.data_ptr(), s=128, stream=s.cuda_stream)
            outs.append((dq, dr, s))
    torch.cuda.synchronize()
    for (dq, dr, _), (_, _, (wq, wr)) in zip(outs, cases * 2):
        assert np.array_equal(np.trim_zeros(dq.cpu().numpy().view(np.uint32), "b"), wq)
        assert np.array_equal(np.trim_zeros(dr.cpu().numpy().view(np.uint32), "b"), wr)
    errs = []

    def worker(k):
        try:
            for i, (a, b, (wq, wr)) in enumerate(cases[k:] + cases[:k]):
                q, r = mmm.divmod(a, b, P, s=64)
                if not (np.array_equal(q, wq) and np.array_equal(r, wr)):
                    dq = np.nonzero(q != wq)[0] if len(q) == len(wq) else np.array([-1])
                    dr = np.nonzero(r != wr)[0] if len(r) == len(wr) else np.array([-1])
                    q2, r2 = mmm.divmod(a, b, P, s=64)  # diagnostics: transient or not
                    again = np.array_equal(q2, wq) and np.array_equal(r2, wr)
                    same_a = np.array_equal(r, a[: len(r)]) if len(r) <= len(a) else None
                    raise AssertionError(f"thread {k} call {i}: divmod differs: q {len(q)}/{len(wq)} at "
                                         f"{dq[:4]}..{dq[-4:]} ({len(dq)}), r {len(r)}/{len(wr)} at "
                                         f"{dr[:4]}..{dr[-4:]} ({len(dr)}); retry ok={again}; "
                                         f"r==a[:nr] {same_a}; q[-66:-62]={q[-66:-62]} want {wq[-66:-62]}; "
                                         f"r[:3]={r[:3]} want {wr[:3]} a[:3]={a[:3]}")
                m, wm = mmm.mul(a[:3000], b[:2000], P), port.mul(a[:3000], b[:2000], P)
                if not np.array_equal(m, wm):
                    dm = np.nonzero(m != wm)[0] if len(m) == len(wm) else np.array([-1])
                    raise AssertionError(f"thread {k}: mul differs at {dm[:4]}..{dm[-4:]} ({len(dm)})")
            mmm.release_scratch()
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    for _ in range(3):
        ts = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    assert not errs, errs
    mmm.release_scratch()
    q, r = mmm.divmod(cases[0][0], cases[0][1], P)
    assert np.array_equal(q, cases[0][2][0])


def test_out_arrays_dirty_and_rejected(cuda_lib, port):
    """out= / q_out= / r_out=: dirty caller buffers (pinned or not) are fully
    overwritten; wrong shape, dtype or layout raises InvalidArgument."""
    import torch
    mmm = cuda_lib
    rng = np.random.default_rng(41)
    A, B = rng.integers(0, P, (5, 600)), rng.integers(0, P, (5, 300))
    B[:, -1] = np.maximum(B[:, -1], 1)
    wantF = np.stack([np.pad(port.mul(A[i], B[i], P), (0, 0)) for i in range(5)]).astype(np.uint32)
    for pinned in (False, True):
        def buf(shape):
            if pinned:
                return torch.full(shape, -7, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
            return np.full(shape, 0xDEADBEEF, dtype=np.uint32)
        F = buf((5, 899))
        assert mmm.mul_batched(A, B, P, out=F) is F
        assert np.array_equal(F, wantF)
        F = buf((5, 899))
        assert np.array_equal(mmm.ntt_mul_batched(A, B, P, out=F), wantF)
        Q, R = buf((5, 301)), buf((5, 299))
        q, r = mmm.divmod_batched(A, B, P, q_out=Q, r_out=R)
        for i in range(5):
            wq, wr = port.divmod(A[i], B[i], P)
            assert np.array_equal(np.trim_zeros(q[i], "b"), wq)
            assert np.array_equal(np.trim_zeros(r[i], "b"), wr)
        f1 = buf((899,))
        v = mmm.mul(A[0], B[0], P, out=f1)
        assert np.shares_memory(v, f1) and np.array_equal(v, wantF[0])
        f2 = buf((899,))
        assert np.array_equal(mmm.ntt_mul(A[0], B[0], P, out=f2), wantF[0])
    for bad in (np.zeros((5, 898), np.uint32), np.zeros((5, 899), np.int64),
                np.zeros((899, 5), np.uint32).T):
        with pytest.raises(mmm.InvalidArgument):
            mmm.mul_batched(A, B, P, out=bad)
    with pytest.raises(mmm.InvalidArgument):
        mmm.mul(A[0], B[0], P, out=np.zeros(10, np.uint32))


def test_default_results_from_the_pinned_pool(cuda_lib, port):
    """out=None on a batched call: results in page-locked memory from the
    library's pool (mmm_cu_host_alloc), every word written, the buffer reused
    once the previous result (and its views) are dropped; mmm_cu_host_free of
    anything else is rejected."""
    import ctypes
    import gc
    mmm = cuda_lib
    rng = np.random.default_rng(43)
    A, B = rng.integers(0, P, (7, 900)), rng.integers(0, P, (7, 500))
    B[:, -1] = np.maximum(B[:, -1], 1)
    want = [port.mul(A[i], B[i], P) for i in range(7)]
    F = mmm.mul_batched(A, B, P)
    assert F.shape == (7, 1399) and all(np.array_equal(F[i], want[i]) for i in range(7))
    addr = F.ctypes.data
    view = F[3]  # keeps the first buffer alive
    del F
    gc.collect()
    G = mmm.mul_batched(A, B, P)  # the first buffer is still held by `view`
    assert G.ctypes.data != addr and np.array_equal(view, want[3])
    del view, G
    gc.collect()
    H = mmm.ntt_mul_batched(A, B, P)
    assert all(np.array_equal(H[i], want[i]) for i in range(7))
    lib = mmm.load()  # a freed buffer comes back for the next request of its size
    size = (37 << 20) + 5
    p1, p2 = ctypes.c_void_p(), ctypes.c_void_p()
    assert lib.mmm_cu_host_alloc(size, ctypes.byref(p1)) == 0 and p1.value
    assert lib.mmm_cu_host_free(p1) == 0
    assert lib.mmm_cu_host_alloc(size, ctypes.byref(p2)) == 0 and p2.value == p1.value
    assert lib.mmm_cu_host_free(p2) == 0
    A2 = rng.integers(0, P, (7, 1000))
    A2[:, -1] = np.maximum(A2[:, -1], 1)
    Q, R = mmm.divmod_batched(A2, B, P)
    for i in range(7):
        wq, wr = port.divmod(A2[i], B[i], P)
        assert np.array_equal(np.trim_zeros(Q[i], "b"), wq)
        assert np.array_equal(np.trim_zeros(R[i], "b"), wr)
    bogus = (ctypes.c_uint32 * 4)()
    assert mmm.load().mmm_cu_host_free(ctypes.addressof(bogus)) == mmm.InvalidArgument.status


def test_large_operands_validated_on_the_device(cuda_lib):
    """Single calls with operands past 2^18 words check canonical coefficients on
    the device (after the copy) and still raise InvalidArgument -- also when the
    bad word sits under trailing zeros that trimming drops below the threshold,
    and ahead of a domain error (validate_coeffs comes first,
    run_util.hpp:24-29)."""
    mmm = cuda_lib
    rng = np.random.default_rng(61)
    big = rng.integers(0, P, 300_000).astype(np.uint32)
    big[-1] = 5
    bad = big.copy()
    bad[12345] = P  # one word equal to p
    small = rng.integers(0, P, 3_000).astype(np.uint32)
    small[-1] = 7
    for fn in (lambda: mmm.mul(bad, small, P), lambda: mmm.mul(small, bad, P),
               lambda: mmm.ntt_mul(bad, small, P), lambda: mmm.divmod(bad, small, P, s=64),
               lambda: mmm.divmod_fast(bad, small, P), lambda: mmm.divmod(big, np.append(small[:-1], P), P)):
        with pytest.raises(mmm.InvalidArgument):
            fn()
    hidden = np.zeros(300_000, np.uint32)  # 1000 words after trimming, 300k before
    hidden[:1000] = rng.integers(0, P, 1000)
    hidden[999] = 3
    hidden[10] = P + 1
    with pytest.raises(mmm.InvalidArgument):
        mmm.mul(hidden, small, P)
    zero_lead = np.append(small[:-1], 0).astype(np.uint32)  # divisor lead 0: a domain error ...
    with pytest.raises(mmm.InvalidArgument):  # ... but the dividend is checked first
        mmm.divmod(bad, zero_lead, P)
    f = mmm.mul(big, small, P)  # the valid operands still go through
    assert f.size == big.size + small.size - 1


def test_last_schedule_reports_the_launches(cuda_lib, port):
    """mmm_cu_last_schedule: the kernels of the thread's last host call (what
    the drop-in's SimReport.kernels and N/L/K are built from)."""
    mmm = cuda_lib
    rng = np.random.default_rng(51)
    a, b = _rand(rng, P, 3000), _rand(rng, P, 1200)
    mmm.gcd(port.mul(a[:500], b[:300], P), b, P)
    sched = mmm.last_schedule()
    assert [k[0] for k in sched] == ["gcd_kernel"] and sched[0][1] >= 2 and sched[0][2] > 0
    mmm.mul(a, b, P)
    sched = mmm.last_schedule()
    assert sched and all(k[0] == "mul_kernel" for k in sched)
    big_a, big_b = _rand(rng, P, 70_000), _rand(rng, P, 33_000)
    mmm.divmod(big_a, big_b, P, s=128)
    assert [k[0] for k in mmm.last_schedule()] == ["div_pipe_kernel"]
    mmm.divmod(big_a, big_b[:1], P)
    assert [k[0] for k in mmm.last_schedule()] == ["div_const_kernel"]
