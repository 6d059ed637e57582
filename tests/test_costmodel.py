"""The restated cost model against the reference's frozen model values
(proj/tests/test_costmodel.cpp) and its rational rendering (rational.cpp)."""
from fractions import Fraction as Q

import pytest

from paper_1402_0264_b200 import costmodel as cm


def test_division_naive_frozen():  # test_costmodel.cpp:13-26
    t = cm.division_cost(cm.NAIVE, 17, 8, l=4, U=4)
    assert (t.W, t.S, t.O, t.N, t.L, t.C) == (180, 30, 400, 20, 10, 23)


def test_division_blocked_frozen():  # test_costmodel.cpp:28-41
    t = cm.division_cost(cm.OPTIMIZED, 17, 8, s=2, U=4)
    assert (t.W, t.S, t.O, t.N, t.L, t.C) == (190, 30, 360, 10, 5, 42)


def test_division_degenerate_and_validation():  # test_costmodel.cpp:43-76
    assert cm.division_cost(cm.NAIVE, 9, 4, l=1, U=2).C == 3 + 5 * 2
    assert cm.division_cost(cm.OPTIMIZED, 9, 4, s=1, U=2).C == 3 + 9 * 2
    for kw in ({"n": 4, "m": 8}, {"n": 4, "m": 0}):
        with pytest.raises(ValueError):
            cm.division_cost(cm.NAIVE, kw["n"], kw["m"], l=4, U=4)
    with pytest.raises(ValueError):
        cm.division_cost(cm.NAIVE, 8, 4, l=0, U=4)
    with pytest.raises(ValueError):
        cm.division_cost(cm.OPTIMIZED, 8, 4, s=0, U=4)
    with pytest.raises(ValueError):
        cm.division_cost(cm.NAIVE, 8, 4, l=4, U=0)


def test_multiplication_frozen():  # test_costmodel.cpp:78-107
    t = cm.multiplication_cost(8, 8, l=4, s=2, U=4)
    assert (t.W, t.S, t.O, t.N, t.L, t.C) == (Q(279, 2), 10, 189, Q(63, 8), 3, 30)
    t = cm.multiplication_cost(8, 8, l=4, s=1, U=4)
    assert (t.S, t.L, t.C, t.W) == (4, 4, 1 + 4 * 4, Q(31, 2) * 8)
    with pytest.raises(ArithmeticError):
        cm.multiplication_cost(8, 6, l=4, s=2, U=4)  # m/s = 3: no halving schedule
    with pytest.raises(ValueError):
        cm.multiplication_cost(8, 8, l=4, s=3, U=4)


def test_gcd_frozen():  # test_costmodel.cpp:124-152
    t = cm.gcd_cost(cm.NAIVE, 8, 8, l=4, U=4)
    assert (t.W, t.S, t.O, t.N, t.L, t.C) == (150, 42, 520, 26, 14, 23)
    t = cm.gcd_cost(cm.OPTIMIZED, 8, 8, s=2, U=4)
    assert (t.W, t.S, t.O, t.N, t.L, t.C) == (Q(3125, 4), 48, 640, 20, 8, 38)


def test_gcd_span_independent_of_s():  # test_costmodel.cpp:154-163
    for n in (8, 64, 1000):
        for s in (2, 3, 7):
            assert cm.gcd_cost(cm.OPTIMIZED, n, n // 2, s=s, U=Q(3, 2)).S == 3 * n + 3 * (n // 2)


def test_frozen_ratios():  # test_costmodel.cpp:205-237
    assert cm.division_time_ratio(4, 128) == Q(2944, 636)
    assert cm.gcd_time_ratio_limit(4, 128) == Q(2944, 576)
    assert cm.multiplication_essential_ratio(4096, 4) == Q(24, 40)
    for n in (8, 64, 4096):
        assert cm.multiplication_time_ratio(n, 1, 4) == 1
    prev = None
    for n in (16, 256, 4096, 1 << 20):  # finite-size gcd ratio decreases to its limit
        r = cm.gcd_time_ratio(n, 4, 128)
        assert r > cm.gcd_time_ratio_limit(4, 128)
        assert prev is None or r < prev
        prev = r


def test_graham_brent_bound():
    assert cm.graham_brent_bound(20, 10, 23, 4) == (Q(20, 4) + 10) * 23
    with pytest.raises(ValueError):
        cm.graham_brent_bound(1, 1, 1, 0)


@pytest.mark.parametrize("v,text", [
    (Q(279, 2), "139.5"), (Q(63, 8), "7.875"), (Q(1, 3), "1/3"), (Q(-5, 4), "-1.25"),
    (Q(-2, 3), "-2/3"), (Q(7), "7"), (Q(1, 20), "0.05"), (None, ""),
])
def test_rendering(v, text):  # rational.cpp:88-112
    assert cm.render(v) == text


def test_csv_column_order():  # report.cpp:40-80
    r = cm.row("division", cm.OPTIMIZED, n=17, m=8, s=2, U=4,
               pred=cm.division_cost(cm.OPTIMIZED, 17, 8, s=2, U=4), T_bound=Q(1, 3))
    text = cm.to_csv([r], extra=("gpu_ms",))
    head, line = text.strip().split("\n")
    assert head.split(",")[:23] == list(cm.REPORT_COLUMNS) and head.endswith(",gpu_ms")
    cells = dict(zip(head.split(","), line.split(",")))
    assert cells["W_pred"] == "190" and cells["T_bound"] == "1/3" and cells["W_meas"] == ""
