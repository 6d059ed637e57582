"""CPU: the C-ABI library loads, exports exactly what include/mmm_cu.h
declares, its host-side functions (field, generator) match the reference,
and compute entry points validate like the reference and fail loudly -- never
fall back to the CPU -- when no GPU is present."""
import os
import re

import numpy as np
import pytest

import paper_1402_0264_b200 as mmm
from helpers import ProductRng, PyRng, digest
import suites

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mmm_cu.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(mmm_\w+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    lib = mmm.load()
    declared = header_symbols()
    assert declared == set(mmm.SIGNATURES), declared ^ set(mmm.SIGNATURES)
    for name in declared:
        assert hasattr(lib, name), name
    out = os.popen(f"nm -D --defined-only {mmm.LIB_PATH}").read()
    exported = set(re.findall(r"\b(mmm_\w+)\b", out))
    assert declared <= exported


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {mmm.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def test_field_validation_like_reference():
    # test_field.cpp:10-22
    for p in (7, 2, 101, 469762049, 2147483647):
        assert mmm.Field(p).p() == p
    for p in (6, 1, 0, -7, 1 << 31, (1 << 31) + 11):
        with pytest.raises(mmm.InvalidArgument):
            mmm.Field(p)


def test_field_inverse_like_reference():
    F = mmm.Field(7)
    assert F.inv(3) == 5 and F.inv(1) == 1 and F.divide(6, 2) == 3
    with pytest.raises(mmm.DomainError):
        mmm.Field(101).inv(0)
    for p in (2, 7, 101, 65537):
        F = mmm.Field(p)
        for a in range(1, min(p, 300)):
            assert F.mul(a, F.inv(a)) == 1
    F = mmm.Field(2147483647)
    assert F.inv(2147483646) == 2147483646


def test_product_generator_is_the_reference_generator(golden_small):
    a, b = ProductRng(2026), PyRng(2026)
    for _ in range(1000):
        assert a.next() == b.next()
    # the first suite replayed through the product generator reproduces the
    # reference's input digests
    cases = golden_small["suites"]["division_sweep"]["cases"]
    from helpers import replay
    for c, g in zip(replay("division_sweep", ProductRng, None), cases):
        assert (digest(c["a"]), digest(c["b"])) == (g["a"], g["b"])


def test_config_inputs_from_product_generator(golden_configs):
    c = suites.cfg1(ProductRng(42))
    assert (digest(c["a"]), digest(c["b"])) == (golden_configs["cfg1"]["a"],
                                                golden_configs["cfg1"]["b"])


def test_validation_errors_before_any_device_work():
    with pytest.raises(mmm.InvalidArgument):
        mmm.mul([1, 2], [3], 6)  # composite modulus
    with pytest.raises(mmm.InvalidArgument):
        mmm.mul([1, 9], [3], 7)  # non-canonical coefficient
    with pytest.raises(mmm.DomainError):
        mmm.divmod([1, 2, 3], [], 7)  # oracle.cpp:52
    with pytest.raises(mmm.DomainError):
        mmm.gcd([], [], 7)  # oracle.cpp:71
    # zero operand: zero product without touching the device (oracle.cpp:9)
    assert mmm.mul([], [1, 2], 7).size == 0
    # deg a < deg b: quotient 0, remainder a (oracle.cpp:55)
    q, r = mmm.divmod([1, 2], [3, 0, 2, 5], 7)
    assert q.size == 0 and r.tolist() == [1, 2]


def test_fanout_validation_before_any_device_work():
    """Fan-out entry points reject an empty or oversized output set, null
    outputs and mismatched q/r sets before touching the device."""
    for outs in ([], [1] * 9, [0]):
        with pytest.raises(mmm.InvalidArgument):
            mmm.mul_range_fanout_dev(7, 1, 2, 1, 2, 0, 3, outs)
        with pytest.raises(mmm.InvalidArgument):
            mmm.mul_batched_fanout_dev(7, 1, 2, 2, 1, 2, 2, 1, outs, 3)
    with pytest.raises(mmm.InvalidArgument):
        mmm.divmod_batched_fanout_dev(7, 1, 3, 3, 1, 2, 2, 1, [1], 2, [1, 2], 1)
    with pytest.raises(mmm.InvalidArgument):  # shape checked too
        mmm.mul_batched_fanout_dev(7, 1, 1, 2, 1, 2, 2, 1, [1], 3)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    for fn in (lambda: mmm.mul([1, 1], [1, 1], 7), lambda: mmm.divmod([1, 2, 0, 1], [1, 1], 7),
               lambda: mmm.gcd([2, 3, 1], [3, 4, 1], 7),
               lambda: mmm.ntt_mul([1, 2], [3, 4], 469762049)):
        with pytest.raises(mmm.CudaError):
            fn()


def test_host_free_rejects_foreign_pointers():
    """mmm_cu_host_free only takes buffers from mmm_cu_host_alloc (no CUDA call
    is made for a foreign pointer, so this runs without a GPU)."""
    import ctypes
    mmm = pytest.importorskip("paper_1402_0264_b200")
    lib = mmm.load()
    bogus = (ctypes.c_uint32 * 4)()
    assert lib.mmm_cu_host_free(ctypes.addressof(bogus)) == mmm.InvalidArgument.status
    assert lib.mmm_cu_host_free(None) == 0
