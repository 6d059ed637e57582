"""GPU parity: every CUDA entry point, called through the C ABI, against the
reference's golden vectors (tests/golden) and the CPU oracle, bit-exact.

Small suites replay the reference's own seeded tests (suites.py) and compare
digests of the GPU results with the digests the unmodified reference
produced; config-scale cases compare with the reference's digests of the
BASELINE configs; size-independent properties cover the rest."""
import numpy as np
import pytest

from helpers import ProductRng, digest, replay
import suites

pytestmark = pytest.mark.gpu

P = suites.P_BENCH
NTT_PRIMES = [469762049, 998244353, 7340033, 12289, 257, 17, 2013265921]  # the last: > 2^30 (exact butterflies)


def _mul_cpu(port):
    return port.mul


# --------------------------------------------------------- frozen cases --
def test_frozen(cuda_lib, golden_small):
    mmm = cuda_lib
    for c in golden_small["frozen"]:
        p, a, b = c["p"], c["a"], c["b"]
        if c["op"] == "mul":
            for s in (1, 2, 4, 8, 16):
                assert mmm.mul(a, b, p, s=s).tolist() == c["f"]
        elif c["op"] == "divmod":
            for s in (1, 2, 3, 4, 8, 64):
                q, r = mmm.divmod(a, b, p, s=s)
                assert (q.tolist(), r.tolist()) == (c["q"], c["r"]), (c, s)
        else:
            for s in (1, 2, 4, 64):
                assert mmm.gcd(a, b, p, s=s).tolist() == c["g"], (c, s)


# ------------------------------------------------------- seeded suites --
@pytest.mark.parametrize("suite", ["mutual_oracle", "divmod_roundtrip", "planted_gcd",
                                   "division_sweep", "multiplication_sweep", "gcd_sweep",
                                   "acceptance", "verify_p7", "verify_p101",
                                   "verify_p469762049"])
def test_suite(cuda_lib, port, golden_small, suite):
    mmm = cuda_lib
    cases = golden_small["suites"][suite]["cases"]
    for c, g in zip(replay(suite, ProductRng, port.mul), cases):
        p, a, b, op = c["p"], c["a"], c["b"], c["op"]
        assert (digest(a), digest(b)) == (g["a"], g["b"])
        if op == "all":      # acceptance_test.cpp:127-209
            s_mul, s_div, s_gcd = c["s_mul"], [c["s_div"]], c["s_gcd"]
        elif op == "verify":  # mmm_cli.cpp:478-520
            s_mul, s_div, s_gcd = [1, 2, 4], [c["s_div"]], [c["s_gcd"]]
        else:
            s_mul = s_div = s_gcd = c.get("s") or [1, 7, 64]
        if "f" in g:
            src = c["am"] if op == "verify" else a
            for s in s_mul:
                assert digest(mmm.mul(src, b, p, s=s)) == g["f"], (suite, s)
        if "q" in g:
            for s in list(s_div) + [64]:
                q, r = mmm.divmod(a, b, p, s=s)
                assert (digest(q), digest(r)) == (g["q"], g["r"]), (suite, s)
        if "g" in g:
            for s in list(s_gcd) + [64]:
                assert digest(mmm.gcd(a, b, p, s=s)) == g["g"], (suite, s)


# ------------------------------------------------------------ edge cases --
def test_edge_shapes(cuda_lib, port):
    mmm = cuda_lib
    rng = np.random.default_rng(11)
    for p in (2, 3, 7, 101, 469762049, 2147483647):
        for na in (1, 2, 3, 31, 32, 33, 129, 1000):
            for nb in (1, 2, 5, 64, 257):
                a = rng.integers(0, p, na)
                b = rng.integers(0, p, nb)
                a[-1] = max(a[-1], 1)
                b[-1] = max(b[-1], 1)
                assert np.array_equal(mmm.mul(a, b, p), port.mul(a, b, p)), (p, na, nb)
                q, r = mmm.divmod(a, b, p, s=16)
                wq, wr = port.divmod(a, b, p)
                assert np.array_equal(q, wq) and np.array_equal(r, wr), (p, na, nb)
                assert np.array_equal(mmm.gcd(a, b, p, s=8), port.gcd(a, b, p)), (p, na, nb)


def test_untrimmed_and_zero_inputs(cuda_lib, port):
    mmm = cuda_lib
    assert mmm.mul([0, 0], [1, 2], 7).size == 0
    assert mmm.mul([1, 2, 0, 0], [3, 0], 7).tolist() == port.mul([1, 2], [3], 7).tolist()
    assert mmm.gcd([3, 0, 2, 5], [], 7).tolist() == port.monic([3, 0, 2, 5], 7).tolist()
    assert mmm.gcd([], [3, 0, 2, 5], 7).tolist() == port.monic([3, 0, 2, 5], 7).tolist()
    q, r = mmm.divmod([1, 2, 0, 1, 0, 0], [1, 1], 7)
    assert (q.tolist(), r.tolist()) == ([3, 6, 1], [5])


def test_degree_drops_small_field(cuda_lib, port):
    """GF(2)/GF(3)/GF(7): many zero heads and multi-step degree drops."""
    mmm = cuda_lib
    rng = np.random.default_rng(5)
    for t in range(300):
        p = (2, 3, 7)[t % 3]
        g = rng.integers(0, p, rng.integers(1, 12))
        g[-1] = 1
        u = rng.integers(0, p, rng.integers(1, 80))
        v = rng.integers(0, p, rng.integers(1, 80))
        a, b = port.mul(g, u, p), port.mul(g, v, p)
        want = port.gcd(a, b, p) if (len(a) or len(b)) else None
        if want is None:
            continue
        for s in (1, 3, 16, 100):
            assert np.array_equal(mmm.gcd(a, b, p, s=s), want), (t, s)
        if len(b):
            wq, wr = port.divmod(a, b, p)
            for s in (1, 5, 32):
                q, r = mmm.divmod(a, b, p, s=s)
                assert np.array_equal(q, wq) and np.array_equal(r, wr)


# --------------------------------------------------------------- NTT ----
def test_ntt_matches_plain(cuda_lib, port):
    mmm = cuda_lib
    rng = np.random.default_rng(3)
    for p in NTT_PRIMES:
        for na, nb in ((1, 1), (2, 3), (5, 1), (100, 28), (1000, 1000), (2048, 2049)):
            if not (p - 1) % (1 << max(2, (na + nb - 2).bit_length())) == 0:
                continue
            a = rng.integers(0, p, na)
            b = rng.integers(0, p, nb)
            assert np.array_equal(mmm.ntt_mul(a, b, p), port.mul(a, b, p)), (p, na, nb)


def _eval_mod(poly, x, p, chunk=1 << 12):
    """poly(x) mod p, vectorised: chunk dot products against x^j, Horner over chunks."""
    poly = np.asarray(poly, dtype=np.int64)
    pw = np.empty(chunk, dtype=np.int64)
    v = 1
    for j in range(chunk):
        pw[j] = v
        v = v * x % p
    X = v  # x^chunk
    n = -(-len(poly) // chunk) * chunk
    padded = np.zeros(n, dtype=np.int64)
    padded[: len(poly)] = poly
    rows = padded.reshape(-1, chunk)
    acc = 0
    for lo in range(rows.shape[0] - 1, -1, -256):  # top chunks first
        blk = rows[max(0, lo - 255): lo + 1]
        inner = ((blk * pw) % p).sum(axis=1) % p
        for val in inner[::-1]:
            acc = (acc * X + int(val)) % p
    return acc


def test_ntt_every_length(cuda_lib):
    """Every transform length the NTT supports (N = 2^2 .. 2^26: every column /
    row template instantiation, both row-length parities) for a lazy prime
    (< 2^30) and an exact one (> 2^30): bit-exact against the GPU schoolbook
    product (itself pinned to the reference) up to N = 2^14, Schwartz-Zippel
    evaluation at two points beyond."""
    mmm = cuda_lib
    rng = np.random.default_rng(26)
    for p in (469762049, 2013265921):
        for logn in range(2, 27):
            n = 1 << logn
            na = n // 2 if logn % 2 else n // 2 - 3
            nb = n - na  # na + nb - 1 = n - 1 -> transform length n
            a = rng.integers(0, p, max(na, 1)).astype(np.uint32)
            b = rng.integers(0, p, max(nb, 1)).astype(np.uint32)
            a[-1] = b[-1] = 1
            f = mmm.ntt_mul(a, b, p)
            if logn <= 14:
                assert np.array_equal(f, mmm.mul(a, b, p)), (p, logn)
            else:
                assert len(f) == len(a) + len(b) - 1, (p, logn)
                for x in (rng.integers(2, p), rng.integers(2, p)):
                    x = int(x)
                    assert _eval_mod(f, x, p) == _eval_mod(a, x, p) * _eval_mod(b, x, p) % p, (p, logn)


def test_ntt_batched_unaligned_rows(cuda_lib):
    """Batched NTT products whose rows are not 16-byte aligned (odd leading
    dimension: the column kernel's scalar-load path) equal the single products."""
    mmm = cuda_lib
    rng = np.random.default_rng(27)
    for na, nb in ((1001, 999), (4097, 31), (3, 2)):
        A = rng.integers(0, P, (5, na)).astype(np.uint32)
        B = rng.integers(0, P, (5, nb)).astype(np.uint32)
        F = mmm.ntt_mul_batched(A, B, P)
        for i in range(5):
            want = mmm.mul(A[i], B[i], P)
            assert np.array_equal(np.trim_zeros(F[i].astype(np.int64), "b"), want), (na, nb, i)


def test_ntt_rejects_unsupported_prime(cuda_lib):
    with pytest.raises(cuda_lib.InvalidArgument):
        cuda_lib.ntt_mul([1, 2, 3], [4, 5], 7)


# ----------------------------------------------------------- batches ----
def test_batched_equal_single(cuda_lib, port):
    mmm = cuda_lib
    rng = np.random.default_rng(9)
    A = rng.integers(0, P, (17, 300)).astype(np.uint32)
    B = rng.integers(1, P, (17, 120)).astype(np.uint32)
    F = mmm.mul_batched(A, B, P)
    Q, R = mmm.divmod_batched(A, B, P, s=32)
    Fn = mmm.ntt_mul_batched(A, B, P)
    for i in range(17):
        want = port.mul(A[i], B[i], P)
        assert np.array_equal(np.trim_zeros(F[i].astype(np.int64), "b"), want)
        assert np.array_equal(np.trim_zeros(Fn[i].astype(np.int64), "b"), want)
        wq, wr = port.divmod(A[i], B[i], P)
        assert np.array_equal(np.trim_zeros(Q[i].astype(np.int64), "b"), wq)
        assert np.array_equal(np.trim_zeros(R[i].astype(np.int64), "b"), wr)


# --------------------------------------------------------- config scale --
def test_cfg1_plain_mult(cuda_lib, golden_configs):
    c = suites.cfg1(ProductRng(42))
    for s in (1, 2, 4, 8, 16):
        assert digest(cuda_lib.mul(c["a"], c["b"], P, s=s)) == golden_configs["cfg1"]["f"], s


def _mul_range(mmm, a, b, k0, k1, s):
    import torch
    da = torch.from_numpy(np.asarray(a, dtype=np.uint32).view(np.int32)).cuda()
    db = torch.from_numpy(np.asarray(b, dtype=np.uint32).view(np.int32)).cuda()
    df = torch.full((max(k1 - k0, 1),), -1, dtype=torch.int32, device="cuda")
    mmm.mul_range_dev(P, da.data_ptr(), len(a), db.data_ptr(), len(b), k0, k1, df.data_ptr(), s=s,
                      stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return df.cpu().numpy().view(np.uint32)[: k1 - k0]


def test_mul_range_slices(cuda_lib, port):
    """Output-range product (the cfg1 shard kernel): every slice, including
    empty, single-word, tile-straddling and whole ranges, equals the oracle's
    product coefficients there; the balanced split reassembles the product."""
    from paper_1402_0264_b200.shard import balanced_output_ranges
    rng = np.random.default_rng(11)
    for na, nb in [(300, 200), (1, 50), (50, 1), (2000, 3000)]:
        a = rng.integers(0, P, na).astype(np.uint32)
        b = rng.integers(0, P, nb).astype(np.uint32)
        full = np.zeros(na + nb - 1, np.int64)
        w = port.mul(a, b, P)
        full[: len(w)] = w
        nf = na + nb - 1
        for k0, k1 in [(0, nf), (0, 1), (nf - 1, nf), (5, 5), (nf // 3, 2 * nf // 3),
                       (min(1023, nf - 1), min(2049, nf))]:
            for s in (1, 8):
                got = _mul_range(cuda_lib, a, b, k0, k1, s)
                assert np.array_equal(got.astype(np.int64), full[k0:k1]), (na, nb, k0, k1, s)
        for world in (2, 3, 8):
            parts = [_mul_range(cuda_lib, a, b, k0, k1, 8)
                     for k0, k1 in balanced_output_ranges(na, nb, world, align=128)]
            assert np.array_equal(np.concatenate(parts).astype(np.int64), full)
    with pytest.raises(cuda_lib.InvalidArgument):
        _mul_range(cuda_lib, a, b, 0, na + nb, 8)


def test_cfg1_sharded_ranges(cuda_lib, golden_configs):
    from paper_1402_0264_b200.shard import balanced_output_ranges
    c = suites.cfg1(ProductRng(42))
    for world in (2, 8):
        f = np.concatenate([_mul_range(cuda_lib, c["a"], c["b"], k0, k1, 8)
                            for k0, k1 in balanced_output_ranges(len(c["a"]), len(c["b"]), world,
                                                                 align=32)])
        assert digest(f) == golden_configs["cfg1"]["f"], world


def test_cfg1_via_ntt(cuda_lib, golden_configs):
    c = suites.cfg1(ProductRng(42))
    assert digest(cuda_lib.ntt_mul(c["a"], c["b"], P)) == golden_configs["cfg1"]["f"]


def test_cfg2_gcd(cuda_lib, port, golden_configs):
    c = suites.cfg2(ProductRng(42), port.mul, port.monic)
    assert (digest(c["a"]), digest(c["b"])) == (golden_configs["cfg2"]["a"],
                                                golden_configs["cfg2"]["b"])
    for s in (8, 32, 64, 128, 256):
        g = cuda_lib.gcd(c["a"], c["b"], P, s=s)
        assert digest(g) == golden_configs["cfg2"]["g"], s
        assert np.array_equal(g, c["g"])


@pytest.mark.parametrize("s", [1, 2, 4, 8, 16, 32, 64, 128, 256, 512])
def test_cfg3_division_sweep(cuda_lib, golden_configs, s):
    c = suites.cfg3(ProductRng(42))
    q, r = cuda_lib.divmod(c["a"], c["b"], P, s=s)
    assert (digest(q), digest(r)) == (golden_configs["cfg3"]["q"], golden_configs["cfg3"]["r"])


def test_cfg3_roundtrip_property(cuda_lib):
    """Size-independent check: q*b + r == a with the GPU's own product."""
    c = suites.cfg3(ProductRng(42))
    q, r = cuda_lib.divmod(c["a"], c["b"], P, s=128)
    qb = cuda_lib.ntt_mul(q, c["b"], P).astype(np.int64)
    qb[: len(r)] = (qb[: len(r)] + r) % P
    assert np.array_equal(qb, np.asarray(c["a"], dtype=np.int64))


def test_cfg4_big_ntt(cuda_lib, golden_configs):
    rng = ProductRng(42)
    c = suites.cfg4_big(rng)
    assert (digest(c["a"]), digest(c["b"])) == (golden_configs["cfg4_big"]["a"],
                                                golden_configs["cfg4_big"]["b"])
    f = cuda_lib.ntt_mul(c["a"], c["b"], P)
    if "f" in golden_configs["cfg4_big"]:
        assert digest(f) == golden_configs["cfg4_big"]["f"]
    # evaluation at random points (Schwartz-Zippel): f(x) == a(x) b(x)
    for x in (3, 123456789, 469762000):
        def ev(poly):
            acc = 0
            for coef in np.asarray(poly, dtype=object)[::-1]:
                acc = (acc * x + int(coef)) % P
            return acc
        assert ev(f) == ev(c["a"]) * ev(c["b"]) % P


def test_cfg4_batch_ntt(cuda_lib, golden_configs):
    rng = ProductRng(42)
    suites.cfg4_big(rng)
    cb = suites.cfg4_batch(rng)
    F = cuda_lib.ntt_mul_batched(cb["A"], cb["B"], P)
    fs = [digest(np.trim_zeros(F[i].astype(np.int64), "b")) for i in range(F.shape[0])]
    assert fs == golden_configs["cfg4_batch"]["f"]


def test_cfg5_batches(cuda_lib, golden_configs):
    c5 = suites.cfg5(ProductRng(42))
    F = cuda_lib.mul_batched(c5["A"], c5["B"], P)
    fs = [digest(np.trim_zeros(F[i].astype(np.int64), "b")) for i in range(F.shape[0])]
    assert fs == golden_configs["cfg5"]["f"]
    Q, R = cuda_lib.divmod_batched(c5["C"], c5["D"], P)
    qs = [digest(np.trim_zeros(Q[i].astype(np.int64), "b")) for i in range(Q.shape[0])]
    rs = [digest(np.trim_zeros(R[i].astype(np.int64), "b")) for i in range(R.shape[0])]
    assert qs == golden_configs["cfg5"]["q"] and rs == golden_configs["cfg5"]["r"]


# ---------------------------------------------- Newton/NTT fast division --
def test_fast_division_frozen_and_suites(cuda_lib, port, golden_small):
    """divmod_fast returns exactly oracle_divmod's (q, r): the frozen GF(7)
    cases and every seeded division suite of the reference's tests."""
    mmm = cuda_lib
    for c in golden_small["frozen"]:
        if c["op"] == "divmod":
            q, r = mmm.divmod_fast(c["a"], c["b"], c["p"])
            assert (q.tolist(), r.tolist()) == (c["q"], c["r"]), c
    for suite in ("mutual_oracle", "divmod_roundtrip", "division_sweep", "acceptance",
                  "verify_p7", "verify_p101", "verify_p469762049"):
        cases = golden_small["suites"][suite]["cases"]
        for c, g in zip(replay(suite, ProductRng, port.mul), cases):
            if "q" in g:
                q, r = mmm.divmod_fast(c["a"], c["b"], c["p"])
                assert (digest(q), digest(r)) == (g["q"], g["r"]), suite


def test_fast_division_edges(cuda_lib, port):
    """Every quotient length around the Newton doubling and the NTT/schoolbook
    switch, constant and monic divisors, p = 2 and primes without 2-adic roots
    (schoolbook products), untrimmed inputs, na < nb and the domain errors."""
    mmm = cuda_lib
    rng = np.random.default_rng(21)
    for p in (2, 7, 101, 469762049, 998244353, 2147483647):
        for na, nb in [(1, 1), (2, 1), (5, 1), (9, 4), (64, 1), (65, 2), (300, 299), (513, 1),
                       (1024, 511), (1100, 512), (2049, 1025), (3000, 700), (700, 3000)]:
            a = rng.integers(0, p, na)
            b = rng.integers(0, p, nb)
            a[-1] = max(a[-1], 1)
            b[-1] = max(b[-1], 1)
            q, r = mmm.divmod_fast(a, b, p)
            wq, wr = port.divmod(a, b, p)
            assert np.array_equal(q, wq) and np.array_equal(r, wr), (p, na, nb)
    q, r = mmm.divmod_fast([1, 2, 0, 1, 0, 0], [1, 1], 7)  # untrimmed dividend
    assert (q.tolist(), r.tolist()) == ([3, 6, 1], [5])
    with pytest.raises(mmm.DomainError):
        mmm.divmod_fast([1, 2, 3], [], 7)
    with pytest.raises(mmm.DomainError):
        mmm.divmod_fast([1, 2, 3], [1, 0], 7)  # zero lead of b, na >= nb


def test_cfg3_fast_division(cuda_lib, golden_configs):
    c = suites.cfg3(ProductRng(42))
    q, r = cuda_lib.divmod_fast(c["a"], c["b"], P)
    assert (digest(q), digest(r)) == (golden_configs["cfg3"]["q"], golden_configs["cfg3"]["r"])


def test_fast_division_roundtrip_at_scale(cuda_lib):
    """2^20 / 2^19 terms (beyond any oracle run): q*b + r == a, deg r < deg b."""
    rng = np.random.default_rng(3)
    a = rng.integers(0, P, (1 << 20) + 3).astype(np.uint32)
    b = rng.integers(0, P, (1 << 19) + 1).astype(np.uint32)
    a[-1] |= 1
    b[-1] |= 1
    q, r = cuda_lib.divmod_fast(a, b, P)
    assert len(q) == len(a) - len(b) + 1 and len(r) < len(b)
    qb = cuda_lib.ntt_mul(q, b, P).astype(np.int64)
    qb[: len(r)] = (qb[: len(r)] + r) % P
    assert np.array_equal(qb, a.astype(np.int64))


# ------------------------------------------ pipelined single-instance division --
@pytest.mark.parametrize("p", [469762049, 101, 7, 2, 2147483647])
def test_division_pipelined_shapes(cuda_lib, port, p):
    """Large single divisions take the pipelined head/bulk schedule (s >= 32,
    S = s rounded to a power of two in [32, 256]); p = 2^31 - 1 falls back to
    the grid schedule.  Quotient lengths that are not multiples of S (short
    last step), remainders shorter than the head window, remainder lengths
    that are not multiples of the bulk block, every S: exactly the oracle."""
    mmm = cuda_lib
    rng = np.random.default_rng(p % 1000)
    for na, nb in [(12000, 6000), (9001, 700), (5000, 4097), (7000, 300), (20000, 19000),
                   (4500, 30)]:
        a = rng.integers(0, p, na)
        b = rng.integers(0, p, nb)
        a[-1] = max(a[-1], 1)
        b[-1] = max(b[-1], 1)
        wq, wr = port.divmod(a, b, p)
        for s in (32, 100, 128, 256, 1000):
            q, r = mmm.divmod(a, b, p, s=s)
            assert np.array_equal(q, wq) and np.array_equal(r, wr), (p, na, nb, s)


@pytest.mark.parametrize("env", ["MMM_DIV_BULK_GLOBAL_B", "MMM_DIV_GRID"])
def test_division_schedule_fallbacks(cuda_lib, port, env, monkeypatch):
    """The pipelined division with the divisor read from L2 per step (the path
    of divisors too large for the bulk CTAs' shared memory) and the grid
    schedule: the same (q, r) as the oracle."""
    monkeypatch.setenv(env, "1")
    rng = np.random.default_rng(77)
    for na, nb in [(12000, 6000), (9001, 700)]:
        a = rng.integers(0, P, na)
        b = rng.integers(0, P, nb)
        a[-1] = max(a[-1], 1)
        b[-1] = max(b[-1], 1)
        wq, wr = port.divmod(a, b, P)
        for s in (32, 128, 256):
            q, r = cuda_lib.divmod(a, b, P, s=s)
            assert np.array_equal(q, wq) and np.array_equal(r, wr), (env, na, nb, s)


# ------------------------------------------------------ sharded four-step NTT --
def test_ntt_sharded_virtual_ranks(cuda_lib, port):
    """The sharded NTT product (phase kernels over column/row slices, block
    exchanges) with W = 1, 2, 4, 8 virtual ranks on one GPU equals the product,
    for several primes and sizes; bad slices are rejected."""
    import torch
    from paper_1402_0264_b200.shard import ntt_mul_virtual
    mmm = cuda_lib
    rng = np.random.default_rng(13)
    st = torch.cuda.current_stream().cuda_stream
    for p, na, nb in [(469762049, 3000, 2000), (998244353, 700, 1300), (7340033, 5000, 5000),
                      (12289, 100, 200), (469762049, 40000, 30000)]:
        a = rng.integers(0, p, na).astype(np.uint32)
        b = rng.integers(0, p, nb).astype(np.uint32)
        want = np.zeros(na + nb - 1, np.int64)
        w = port.mul(a, b, p) if na * nb <= 4e7 else mmm.mul(a, b, p).astype(np.int64)
        want[: len(w)] = w
        da = torch.from_numpy(a.view(np.int32)).cuda()
        db = torch.from_numpy(b.view(np.int32)).cuda()
        for world in (1, 2, 4, 8):
            n1, n2 = mmm.ntt_shape(p, na + nb - 1)
            if n1 % world or n2 % (4 * world):
                continue
            f = ntt_mul_virtual(mmm, p, da, na, db, nb, world, st).cpu().numpy()
            assert np.array_equal(f, want), (p, na, nb, world)
    with pytest.raises(mmm.InvalidArgument):  # column slice not a multiple of 4
        mmm.ntt_phase_dev(469762049, 0, da.data_ptr(), na, db.data_ptr(), nb, 2, 4, 0, 0, 0, st)


def test_cfg4_big_sharded_virtual(cuda_lib, golden_configs):
    import torch
    from paper_1402_0264_b200.shard import ntt_mul_virtual
    c = suites.cfg4_big(ProductRng(42))
    if "f" not in golden_configs["cfg4_big"]:
        pytest.skip("no golden product digest")
    da = torch.from_numpy(np.asarray(c["a"], np.uint32).view(np.int32)).cuda()
    db = torch.from_numpy(np.asarray(c["b"], np.uint32).view(np.int32)).cuda()
    st = torch.cuda.current_stream().cuda_stream
    for world in (2, 8):
        f = ntt_mul_virtual(cuda_lib, P, da, len(c["a"]), db, len(c["b"]), world, st)
        assert digest(f.cpu().numpy()) == golden_configs["cfg4_big"]["f"], world


# ------------------------------------- fan-out outputs (fused all-gather) --
def _dev_u32(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint32).view(np.int32)).cuda()


def test_fanout_mul_range_virtual_ranks(cuda_lib, port):
    """W virtual ranks on one GPU: rank r computes its balanced output range and
    stores it into all W full-product buffers (the symmetric-memory all-gather
    fused into the epilogue); every buffer ends up the whole product, for the
    direct-store and the split-k (finalize) paths."""
    import torch
    from paper_1402_0264_b200.shard import balanced_output_ranges
    rng = np.random.default_rng(21)
    for na, nb in [(3000, 2000), (16384, 16384), (70, 1)]:
        a = rng.integers(0, P, na).astype(np.uint32)
        b = rng.integers(0, P, nb).astype(np.uint32)
        want = np.zeros(na + nb - 1, np.int64)
        w = port.mul(a, b, P)
        want[: len(w)] = w
        da, db = _dev_u32(a), _dev_u32(b)
        for world in (1, 3, 8):
            bufs = [torch.full((na + nb - 1,), -1, dtype=torch.int32, device="cuda")
                    for _ in range(world)]
            for k0, k1 in balanced_output_ranges(na, nb, world, align=32):
                cuda_lib.mul_range_fanout_dev(P, da.data_ptr(), na, db.data_ptr(), nb, k0, k1,
                                              [t.data_ptr() + 4 * k0 for t in bufs], s=4)
            torch.cuda.synchronize()
            for t in bufs:
                assert np.array_equal(t.cpu().numpy().view(np.uint32).astype(np.int64), want), \
                    (na, nb, world)


def test_fanout_batches_virtual_ranks(cuda_lib, port):
    """cfg5-shaped batches split over W virtual ranks: each rank's rows of the
    product and quotient/remainder batches land in every rank's full buffers."""
    import torch
    from paper_1402_0264_b200.shard import shard_range
    rng = np.random.default_rng(22)
    count, na, nb, nd = 10, 300, 200, 150
    A = rng.integers(0, P, (count, na)).astype(np.uint32)
    B = rng.integers(0, P, (count, nb)).astype(np.uint32)
    A[:, -1] |= 1
    B[:, -1] |= 1
    D = rng.integers(0, P, (count, nd)).astype(np.uint32)
    D[:, -1] |= 1
    dA, dB, dD = _dev_u32(A), _dev_u32(B), _dev_u32(D)
    nf, nq, nr = na + nb - 1, na - nd + 1, nd - 1
    for world in (1, 2, 3):
        F = [torch.full((count, nf), -1, dtype=torch.int32, device="cuda") for _ in range(world)]
        Q = [torch.full((count, nq), -1, dtype=torch.int32, device="cuda") for _ in range(world)]
        R = [torch.full((count, nr), -1, dtype=torch.int32, device="cuda") for _ in range(world)]
        for r in range(world):
            i0, i1 = shard_range(count, world, r)
            if i1 <= i0:
                continue
            cuda_lib.mul_batched_fanout_dev(P, dA.data_ptr() + 4 * i0 * na, na, na,
                                            dB.data_ptr() + 4 * i0 * nb, nb, nb, i1 - i0,
                                            [t.data_ptr() + 4 * i0 * nf for t in F], nf, s=8)
            cuda_lib.divmod_batched_fanout_dev(P, dA.data_ptr() + 4 * i0 * na, na, na,
                                               dD.data_ptr() + 4 * i0 * nd, nd, nd, i1 - i0,
                                               [t.data_ptr() + 4 * i0 * nq for t in Q], nq,
                                               [t.data_ptr() + 4 * i0 * nr for t in R], nr, s=64)
        torch.cuda.synchronize()
        for i in range(count):
            wf = port.mul(A[i], B[i], P)
            wq, wr = port.divmod(A[i], D[i], P)
            for q in range(world):
                f = F[q][i].cpu().numpy().view(np.uint32).astype(np.int64)
                assert np.array_equal(np.trim_zeros(f, "b"), wf), (world, q, i)
                assert np.array_equal(Q[q][i].cpu().numpy().view(np.uint32).astype(np.int64), wq)
                rr = R[q][i].cpu().numpy().view(np.uint32).astype(np.int64)
                assert np.array_equal(np.trim_zeros(rr, "b"), wr), (world, q, i)


def test_fanout_copy(cuda_lib):
    """The peer push kernel: every destination equals the source, for aligned
    (vector) and unaligned (scalar) pointers and ragged lengths."""
    import torch
    rng = np.random.default_rng(23)
    for n in (0, 1, 5, 4096, 100003):
        src = _dev_u32(rng.integers(0, P, n + 3).astype(np.uint32))
        for off in (0, 1):
            dst = [torch.full((n + 8,), -1, dtype=torch.int32, device="cuda") for _ in range(3)]
            cuda_lib.fanout_copy_dev(src.data_ptr() + 4 * off, n, [t.data_ptr() + 4 * off for t in dst])
            torch.cuda.synchronize()
            for t in dst:
                assert torch.equal(t[off: off + n], src[off: off + n]), (n, off)
                assert int((t[off + n:] == -1).sum()) == n + 8 - off - n
