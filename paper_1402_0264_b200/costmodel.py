"""The paper's closed-form cost model, restated for the model-vs-measured s
sweep (`tools/s_sweep.py` prints it beside B200 timings).

Each application model yields the six exact quantities of the paper's abstract
machine (proj/include/mmm/costmodel.hpp:22-29): work W, span S, transfer
overhead O, thread blocks N, block-DAG critical path L and the largest
per-block charge C; the running-time estimate is the Graham-Brent bound
(N/P + L)*C (proj/src/metrics.cpp:94-97).  Rationals are `fractions.Fraction`
and render like the reference's Rat (decimal when the reduced denominator is
2^a 5^b, else num/den: proj/src/rational.cpp:88-112).  Rows serialise in
ReportRow's column order (proj/src/report.cpp:40-80) so CSV tooling built for
the reference reads them; measured-on-B200 columns are appended after it.

Host-side analysis only: nothing here touches the GPU or the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction as Q
from typing import Iterable, Optional

NAIVE, OPTIMIZED = "naive", "optimized"


@dataclass(frozen=True)
class CostTuple:
    W: Q
    S: Q
    O: Q
    N: Q
    L: Q
    C: Q


def _need(ok: bool, msg: str):
    if not ok:
        raise ValueError(msg)


def ilog2_exact(v: int) -> int:
    """log2 of a positive power of two, else ArithmeticError (the reference's
    std::domain_error; rational.cpp:116-123)."""
    if v < 1 or v & (v - 1):
        raise ArithmeticError(f"log2: {v} is not a power of two")
    return v.bit_length() - 1


def division_cost(variant: str, n: int, m: int, *, l: int = 1, s: int = 1,
                  U=Q(2)) -> CostTuple:
    """Long division of an n-term by an m-term polynomial, mu = n - m + 1
    quotient terms (costmodel.cpp:26-54)."""
    _need(1 <= m <= n, "division cost model requires n >= m >= 1")
    U = Q(U)
    _need(U > 0, "division cost model requires U > 0")
    mu, m_ = Q(n - m + 1), Q(m)
    if variant == NAIVE:
        _need(l >= 1, "division cost model requires l >= 1")
        l_ = Q(l)
        return CostTuple(W=mu * m_ * (2 * l_ + 1) / l_, S=3 * mu, O=5 * mu * m_ * U / l_,
                         N=mu * m_ / l_, L=mu, C=3 + 5 * U)
    _need(s >= 1, "division cost model requires s >= 1")
    s_ = Q(s)
    return CostTuple(W=mu * m_ * (9 * s_ + 1) / (4 * s_), S=3 * mu,
                     O=9 * mu * m_ * U / (2 * s_ * s_), N=mu * m_ / (2 * s_ * s_),
                     L=mu / s_, C=3 * s_ + 9 * U)


def multiplication_cost(n: int, m: int, *, l: int, s: int, U=Q(2)) -> CostTuple:
    """Long multiplication with s x s thread tiles and a halving addition tree
    over m/s partial rows; delta = n + s - 1 columns (costmodel.cpp:56-80)."""
    _need(n >= 1 and m >= 1, "multiplication cost model requires n, m >= 1")
    _need(l >= 1, "multiplication cost model requires l >= 1")
    _need(1 <= s <= m and m % s == 0, "multiplication cost model requires s | m")
    U = Q(U)
    _need(U > 0, "multiplication cost model requires U > 0")
    k = ilog2_exact(m // s)
    n_, m_, l_, s_ = Q(n), Q(m), Q(l), Q(s)
    delta = n_ + s_ - 1
    return CostTuple(W=(2 * m_ - Q(1, 2)) * delta, S=2 * s_ * s_ + s_ * k - s_,
                     O=delta * (5 * m_ * s_ + 2 * m_ - 3 * s_ * s_) * U / (s_ * s_ * l_),
                     N=delta * (2 * m_ - s_) / (s_ * s_ * l_), L=Q(k + 1),
                     C=s_ * (2 * s_ - 1) + 2 * U * (s_ + 1))


def gcd_cost(variant: str, n: int, m: int, *, l: int = 1, s: int = 1, U=Q(2)) -> CostTuple:
    """Euclidean gcd of an n-term and an m-term polynomial (costmodel.cpp:82-110)."""
    _need(1 <= m <= n, "gcd cost model requires n >= m >= 1")
    U = Q(U)
    _need(U > 0, "gcd cost model requires U > 0")
    n_, m_ = Q(n), Q(m)
    if variant == NAIVE:
        _need(l >= 1, "gcd cost model requires l >= 1")
        l_ = Q(l)
        return CostTuple(W=m_ * (2 * n_ * l_ + n_ + l_ - 1) / l_, S=3 * (m_ + n_ - 2),
                         O=5 * m_ * U * (n_ + l_ + 1) / l_, N=m_ * (n_ + l_ + 1) / l_,
                         L=m_ + n_ - 2, C=3 + 5 * U)
    _need(s >= 1, "gcd cost model requires s >= 1")
    s_ = Q(s)
    W = ((Q(9, 4) + 6 / s_) * m_ * m_
         + (9 * n_ / 2 + n_ / (2 * s_) + Q(87, 8) * s_ + Q(23, 2)) * m_
         - Q(345, 16) * s_ * s_ - Q(77, 4) * s_)
    return CostTuple(W=W, S=3 * n_ + 3 * m_, O=8 * m_ * U * (n_ + s_) / (s_ * s_),
                     N=m_ * n_ / (s_ * s_) + m_ / s_, L=n_ / s_ + m_ / s_, C=3 * s_ + 8 * U)


def graham_brent_bound(N, L, C, P: int) -> Q:
    """(N/P + L) * C (metrics.cpp:94-97)."""
    _need(P >= 1, "graham_brent_bound: P must be >= 1")
    return (Q(N) / P + Q(L)) * Q(C)


# --- naive / optimized time-estimate ratios (costmodel.cpp:141-210) ----------
def division_time_ratio(U, Z) -> Q:
    U, Z = Q(U), Q(Z)
    _need(U > 0 and Z > 0, "division time ratio requires U, Z > 0")
    return (3 + 5 * U) * Z / (3 * (Z + 21 * U))


def gcd_time_ratio(n, U, Z) -> Q:
    n, U, Z = Q(n), Q(U), Q(Z)
    _need(n > 0 and U > 0 and Z > 0, "gcd time ratio requires n, U, Z > 0")
    return (6 * n - 2 + Z) * (3 + 5 * U) * Z / ((18 * n + Z) * (Z + 16 * U))


def gcd_time_ratio_limit(U, Z) -> Q:
    U, Z = Q(U), Q(Z)
    _need(U > 0 and Z > 0, "gcd time ratio requires U, Z > 0")
    return (3 + 5 * U) * Z / (3 * (Z + 16 * U))


def multiplication_essential_ratio(n: int, s: int) -> Q:
    _need(1 <= s < n and n % s == 0, "multiplication essential ratio requires s | n, s < n")
    return Q(2 * ilog2_exact(n), s * ilog2_exact(n // s))


def multiplication_time_ratio(n: int, s: int, U) -> Q:
    _need(1 <= s <= n and n % s == 0, "multiplication time ratio requires s | n")
    U = Q(U)
    _need(U > 0, "multiplication time ratio requires U > 0")
    N_, S_ = Q(n), Q(s)
    lg_n, lg_ns = ilog2_exact(n), ilog2_exact(n // s)
    return ((N_ * lg_n + 3 * N_ - 1) * (1 + 4 * U)
            / ((N_ * lg_ns + 3 * N_ - S_) * (2 * U * S_ + 2 * U + 2 * S_ * S_ - S_)))


# --- ReportRow serialisation --------------------------------------------------
REPORT_COLUMNS = (
    "app", "variant", "n", "m", "l", "s", "U", "Z",
    "W_meas", "W_pred", "S_meas", "S_pred", "O_meas", "O_pred",
    "N_meas", "N_pred", "L_meas", "L_pred", "C_meas", "C_pred",
    "K", "T_bound", "ratio",
)  # report.cpp:40-80, in order


def render(v) -> str:
    """Canonical rendering of a rational (rational.cpp:88-112); None -> ''."""
    if v is None:
        return ""
    if isinstance(v, str):
        return v
    if isinstance(v, int):
        return str(v)
    q = Q(v)
    if q.denominator == 1:
        return str(q.numerator)
    d, twos, fives = q.denominator, 0, 0
    while d % 2 == 0:
        d //= 2
        twos += 1
    while d % 5 == 0:
        d //= 5
        fives += 1
    if d != 1:
        return f"{q.numerator}/{q.denominator}"
    k = max(twos, fives)
    scaled = abs(q.numerator) * 10 ** k // q.denominator
    ip, fp = divmod(scaled, 10 ** k)
    frac = str(fp).rjust(k, "0").rstrip("0")
    out = ("-" if q < 0 else "") + str(ip)
    return out + ("." + frac if frac else "")


def row(app: str, variant: str, *, n=None, m=None, l=None, s=None, U=None, Z=None,
        pred: Optional[CostTuple] = None, meas: Optional[dict] = None, K=None,
        T_bound=None, ratio=None) -> dict:
    """One ReportRow as a column -> value dict (values rendered at to_csv)."""
    r = dict.fromkeys(REPORT_COLUMNS)
    r.update(app=app, variant=variant, n=n, m=m, l=l, s=s, U=U, Z=Z, K=K,
             T_bound=T_bound, ratio=ratio)
    if pred is not None:
        for f in "WSONLC":
            r[f + "_pred"] = getattr(pred, f)
    for k, v in (meas or {}).items():
        r[k + "_meas"] = v
    return r


def to_csv(rows: Iterable[dict], extra: tuple = ()) -> str:
    """Header plus one line per row: ReportRow columns, then `extra` columns."""
    cols = REPORT_COLUMNS + tuple(extra)
    lines = [",".join(cols)]
    for r in rows:
        lines.append(",".join(render(r.get(c)) for c in cols))
    return "\n".join(lines) + "\n"
