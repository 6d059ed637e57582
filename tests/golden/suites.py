"""Seeded parity suites restated from the reference's own tests.

Each generator reproduces, draw for draw, the input stream of one reference
test (same seed, same ``rng() % k`` size draws, same ``random_poly`` calls in
the same order), so the golden outputs recorded by ``make_golden.py`` from the
reference build are the reference's own answers on the reference's own
instances.  ``rng`` is any object with ``next() -> int`` (raw mt19937_64
output) and ``random_poly(terms, p) -> np.ndarray``.

Cases are dicts: {"suite", "op", "p", "a", "b", ...params}; op is one of
"mul", "divmod", "gcd".  Product-of-planted-factor inputs are built with the
CPU oracle passed as ``mul`` (the reference's tests do the same).
"""
from __future__ import annotations

from typing import Callable, Iterator

import numpy as np


def _pick(rng, lo: int, hi: int) -> int:
    """acceptance_test.cpp:55-57 / mmm_cli.cpp:452-454."""
    return lo + rng.next() % (hi - lo + 1)


def mutual_oracle(rng, mul) -> Iterator[dict]:
    """test_poly_oracle.cpp:105-119 (seed 2026): 1000 products over GF(7)/GF(101)."""
    for t in range(1000):
        p = 7 if t % 2 == 0 else 101
        n = 1 + rng.next() % 20
        m = 1 + rng.next() % 20
        a = rng.random_poly(n, p)
        b = rng.random_poly(m, p)
        yield dict(suite="mutual_oracle", op="mul", p=p, a=a, b=b)


def divmod_roundtrip(rng, mul) -> Iterator[dict]:
    """test_poly_oracle.cpp:80-95 (seed 123)."""
    for p in (7, 101):
        for _ in range(80):
            m = 1 + rng.next() % 24
            n = m + rng.next() % 24
            a = rng.random_poly(n, p)
            b = rng.random_poly(m, p)
            yield dict(suite="divmod_roundtrip", op="divmod", p=p, a=a, b=b)


def planted_gcd(rng, mul) -> Iterator[dict]:
    """test_poly_oracle.cpp:148-171 (seed 5150, GF(101))."""
    p = 101
    for _ in range(60):
        g = rng.random_poly(1 + rng.next() % 6, p)
        u = rng.random_poly(1 + rng.next() % 10, p)
        v = rng.random_poly(1 + rng.next() % 10, p)
        yield dict(suite="planted_gcd", op="gcd", p=p, a=mul(g, u, p), b=mul(g, v, p), g=g)


def division_sweep(rng, mul) -> Iterator[dict]:
    """test_division.cpp:83-109 (seed 424242), s in {1,2,3,4,8} + naive l=4."""
    for p in (7, 101):
        for _ in range(20):
            m = 1 + rng.next() % 20
            n = m + rng.next() % 30
            a = rng.random_poly(n, p)
            b = rng.random_poly(m, p)
            yield dict(suite="division_sweep", op="divmod", p=p, a=a, b=b, s=[1, 2, 3, 4, 8])


def multiplication_sweep(rng, mul) -> Iterator[dict]:
    """test_multiplication.cpp:51-70 (seed 1337), s in {1,2,3,4,8} x l in {1,4,16}."""
    for p in (7, 101):
        for _ in range(15):
            n = 1 + rng.next() % 40
            m = 1 + rng.next() % 40
            a = rng.random_poly(n, p)
            b = rng.random_poly(m, p)
            yield dict(suite="multiplication_sweep", op="mul", p=p, a=a, b=b, s=[1, 2, 3, 4, 8],
                       l=[1, 4, 16])


def gcd_sweep(rng, mul) -> Iterator[dict]:
    """test_gcd.cpp:99-123 (seed 4242): random pairs, then planted factors."""
    for p in (7, 101):
        for _ in range(12):
            ta = 1 + rng.next() % 24
            tb = 1 + rng.next() % 24
            if ta < tb:
                ta, tb = tb, ta
            a = rng.random_poly(ta, p)
            b = rng.random_poly(tb, p)
            yield dict(suite="gcd_sweep", op="gcd", p=p, a=a, b=b, s=[2, 4, 8])
        for _ in range(8):
            g = rng.random_poly(5, p)
            a = mul(g, rng.random_poly(9, p), p)
            b = mul(g, rng.random_poly(7, p), p)
            if len(a) < len(b):
                a, b = b, a
            yield dict(suite="gcd_sweep_planted", op="gcd", p=p, a=a, b=b, s=[2])


def acceptance(rng_factory: Callable[[int], object], mul) -> Iterator[dict]:
    """acceptance_test.cpp:122-209: seeds 20260819+p, 200 trials, sizes <= 256."""
    for p in (7, 101):
        rng = rng_factory(20260819 + p)
        for trial in range(200):
            m = 256 if trial == 0 else _pick(rng, 1, 256)
            n = 256 if trial == 0 else _pick(rng, m, 256)
            a = rng.random_poly(n, p)
            b = rng.random_poly(m, p)
            l = _pick(rng, 1, 8)
            s_div = _pick(rng, 1, 8)
            yield dict(suite="acceptance", op="all", p=p, a=a, b=b, l=l, s_div=s_div,
                       s_mul=[1, 2, 4, 8], s_gcd=[2, 4, 8, 16])


def verify(rng, p: int, trials: int = 200, max_n: int = 64, Z: int = 1024) -> Iterator[dict]:
    """mmm_cli.cpp:456-528 (`mmm verify`, default seed 42)."""
    for _ in range(trials):
        m = _pick(rng, 1, max_n)
        n = _pick(rng, m, max_n)
        nm = _pick(rng, 1, max_n)
        l = _pick(rng, 1, min(8, Z // 2))
        s_div = _pick(rng, 1, min(8, Z // 7))
        s_gcd = _pick(rng, 2, min(8, Z // 6))
        a = rng.random_poly(n, p)
        b = rng.random_poly(m, p)
        am = rng.random_poly(nm, p)
        yield dict(suite=f"verify_p{p}", op="verify", p=p, a=a, b=b, am=am, l=l, s_div=s_div,
                   s_gcd=s_gcd)


# Frozen GF(7)/GF(101) instances written out in the reference's tests.
FROZEN = [
    # test_poly_oracle.cpp:55-62, test_division.cpp:29-46
    dict(op="divmod", p=7, a=[1, 2, 0, 1], b=[1, 1], q=[3, 6, 1], r=[5]),
    # test_division.cpp:48-53 (self-division)
    dict(op="divmod", p=101, a=[3, 0, 7, 1], b=[3, 0, 7, 1], q=[1], r=[]),
    # test_poly_oracle.cpp:64-77 (edge shapes)
    dict(op="divmod", p=7, a=[3, 0, 2, 5], b=[3, 0, 2, 5], q=[1], r=[]),
    dict(op="divmod", p=7, a=[1, 2], b=[3, 0, 2, 5], q=[], r=[1, 2]),
    # test_division.cpp:68-81 (interior zeros / degree drops)
    dict(op="divmod", p=7, a=[1, 0, 0, 0, 0, 1], b=[1, 0, 1], q=None, r=None),
    # test_poly_oracle.cpp:97-103, test_multiplication.cpp:28-34
    dict(op="mul", p=7, a=[1, 1], b=[1, 1], f=[1, 2, 1]),
    dict(op="mul", p=7, a=[3], b=[2, 5, 1], f=[6, 1, 3]),
    dict(op="mul", p=7, a=[2, 5, 1], b=[1], f=[2, 5, 1]),
    dict(op="mul", p=7, a=[2, 5, 1], b=[], f=[]),
    # test_poly_oracle.cpp:129-133, test_gcd.cpp:39-46
    dict(op="gcd", p=7, a=[2, 3, 1], b=[3, 4, 1], g=[1, 1]),
    # test_poly_oracle.cpp:135-146 (zero operands)
    dict(op="gcd", p=7, a=[3, 0, 2, 5], b=[], g=None),
    dict(op="gcd", p=7, a=[], b=[3, 0, 2, 5], g=None),
    # test_gcd.cpp:48-65 (divisor pair, identical operands, coprime)
    dict(op="gcd", p=7, a="mul:2,4,6|1,0,5,1", b=[2, 4, 6], g=None),
    dict(op="gcd", p=7, a="mul:2,4,6|1,0,5,1", b="mul:2,4,6|1,0,5,1", g=None),
    dict(op="gcd", p=7, a="mul:1,1|1,1", b=[2, 1], g=[1]),
    # test_gcd.cpp:67-80 (two constants)
    dict(op="gcd", p=101, a=[42], b=[9], g=[1]),
    # test_poly_oracle.cpp:173-179 (coprime linear factors over GF(101))
    dict(op="gcd", p=101, a="mul:100,1|99,1", b="mul:98,1|97,1", g=[1]),
]


def materialise(v, p, mul):
    """Expand the "mul:x|y" shorthand of FROZEN into a coefficient array."""
    if isinstance(v, str):
        x, y = v[4:].split("|")
        return mul(np.array([int(t) for t in x.split(",")]), np.array([int(t) for t in y.split(",")]),
                   p)
    return np.array(v, dtype=np.int64)


# Config-scale inputs (BASELINE.json configs): one fresh
# mt19937_64(42) stream per config, draws in the order listed.
P_BENCH = 469762049


def cfg1(rng):
    """2^14 x 2^14 plain multiplication."""
    return dict(a=rng.random_poly(1 << 14, P_BENCH), b=rng.random_poly(1 << 14, P_BENCH))


def cfg2(rng, mul, monic):
    """GCD of g*u, g*v with g monic of degree 2^12, deg u = 2^13, deg v = 2^13-1."""
    g = monic(rng.random_poly((1 << 12) + 1, P_BENCH), P_BENCH)
    u = rng.random_poly((1 << 13) + 1, P_BENCH)
    v = rng.random_poly(1 << 13, P_BENCH)
    return dict(a=mul(g, u, P_BENCH), b=mul(g, v, P_BENCH), g=g)


def cfg3(rng):
    """Division of degree 2^16 by degree 2^15."""
    return dict(a=rng.random_poly((1 << 16) + 1, P_BENCH), b=rng.random_poly((1 << 15) + 1, P_BENCH))


def cfg4_big(rng):
    """2^20-term x 2^20-term product (NTT length 2^21)."""
    return dict(a=rng.random_poly(1 << 20, P_BENCH), b=rng.random_poly(1 << 20, P_BENCH))


def cfg4_batch(rng, count=256, terms=1 << 15):
    """256 independent 2^15 x 2^15 products (NTT length 2^16); same stream
    after cfg4_big's two draws when ``rng`` is shared."""
    A = np.empty((count, terms), dtype=np.int64)
    B = np.empty((count, terms), dtype=np.int64)
    for i in range(count):
        A[i] = rng.random_poly(terms, P_BENCH)
        B[i] = rng.random_poly(terms, P_BENCH)
    return dict(A=A, B=B)


def cfg5(rng, count=4096, terms=4096):
    """4096 products 4096x4096, then 4096 divisions 8192 by 4096 terms."""
    A = np.empty((count, terms), dtype=np.int64)
    B = np.empty((count, terms), dtype=np.int64)
    for i in range(count):
        A[i] = rng.random_poly(terms, P_BENCH)
        B[i] = rng.random_poly(terms, P_BENCH)
    Cd = np.empty((count, 2 * terms), dtype=np.int64)
    D = np.empty((count, terms), dtype=np.int64)
    for i in range(count):
        Cd[i] = rng.random_poly(2 * terms, P_BENCH)
        D[i] = rng.random_poly(terms, P_BENCH)
    return dict(A=A, B=B, C=Cd, D=D)
