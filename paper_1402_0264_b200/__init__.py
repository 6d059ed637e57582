"""paper_1402_0264_b200 -- B200 (sm_100a) polynomial arithmetic over Z/pZ.

Python face of the C ABI in ``include/mmm_cu.h`` (library
``paper_1402_0264_b200/lib/libmmm_cu.so``, built by ``__graft_entry__.build()``
or ``make -C paper_1402_0264_b200/csrc``).  The functions mirror the
reference's oracle-style entry points (proj/include/mmm/oracle.hpp) and its
blocked kernel programs (run_multiplication / run_division / run_gcd), with
the same argument meaning and error behaviour:

    mul(a, b, p, s=0)            == oracle_mul        (oracle.cpp:8-15)
    divmod(a, b, p, s=64)        == oracle_divmod     (oracle.cpp:51-67)
    gcd(a, b, p, s=64)           == oracle_gcd        (oracle.cpp:69-78)
    ntt_mul(a, b, p)             == oracle_mul        (product uniqueness)
    Field(p), random_poly(rng, terms, F)              (field.cpp, poly.cpp)

The program parameter s: s >= 1 runs the paper's s-parameterised CUDA-core
kernel (register tile / heads per step / steps per matrix batch); s = 0 (the
default for products and batched divisions) lets the library pick, which for
large products and cfg5-sized batches is the integer tensor core.

Polynomials are 1-D numpy arrays of canonical residues, ascending, trimmed
(the zero polynomial is an empty array).  Errors raise ``InvalidArgument``
(std::invalid_argument), ``DomainError`` (std::domain_error) or ``CudaError``.
There is no CPU fallback: without the CUDA library or a GPU, compute calls
raise.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from typing import Optional

import numpy as np

__all__ = [
    "LIB_PATH", "load", "MmmError", "InvalidArgument", "DomainError", "CudaError", "SimError",
    "Field", "Rng", "random_poly", "mul", "divmod", "gcd", "ntt_mul", "mul_batched",
    "divmod_batched", "ntt_mul_batched", "mul_dev", "mul_range_dev", "divmod_dev", "gcd_dev",
    "divmod_fast", "divmod_fast_dev", "ntt_shape", "ntt_phase_dev",
    "ntt_mul_dev",
    "mul_batched_dev", "divmod_batched_dev", "ntt_mul_batched_dev", "launch_count",
    "mul_batched_multi", "divmod_batched_multi", "ntt_mul_batched_multi",
    "mul_batched_multi_dev", "divmod_batched_multi_dev", "ntt_mul_batched_multi_dev",
    "release_scratch", "last_schedule",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MMM_CU_LIB") or os.path.join(HERE, "lib", "libmmm_cu.so")


class MmmError(RuntimeError):
    status = -1


class InvalidArgument(MmmError, ValueError):
    status = 1


class DomainError(MmmError, ArithmeticError):
    status = 2


class CudaError(MmmError):
    status = 3


class SimError(MmmError):
    status = 5


_ERR = {1: InvalidArgument, 2: DomainError, 3: CudaError, 4: MmmError, 5: SimError}

_U32P = C.POINTER(C.c_uint32)
_I64P = C.POINTER(C.c_int64)
_I32P = C.POINTER(C.c_int32)


class KernelRec(C.Structure):
    """mmm_kernel_rec (include/mmm_cu.h)."""
    _fields_ = [("name", C.c_char * 40), ("blocks", C.c_int64), ("threads", C.c_int32)]
_I64 = C.c_int64
_VP = C.c_void_p

# name -> (restype, argtypes); the exact set include/mmm_cu.h declares.
SIGNATURES = {
    "mmm_last_error": (C.c_char_p, []),
    "mmm_version": (C.c_int, []),
    "mmm_cu_launch_count": (C.c_uint64, []),
    "mmm_cu_release_scratch": (C.c_int, []),
    "mmm_cu_last_schedule": (C.c_int, [C.POINTER(KernelRec), C.c_int32, _I32P]),
    "mmm_cu_release_all": (C.c_int, []),
    "mmm_cu_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "mmm_cu_host_free": (C.c_int, [_VP]),
    "mmm_field_check": (C.c_int, [_I64]),
    "mmm_field_inv": (C.c_int, [_I64, _I64, _I64P]),
    "mmm_rng_create": (_VP, [C.c_uint64]),
    "mmm_rng_destroy": (None, [_VP]),
    "mmm_rng_next": (C.c_uint64, [_VP]),
    "mmm_random_poly": (C.c_int, [_VP, _I64, _I64, _U32P]),
    "mmm_cu_mul": (C.c_int, [_I64, _U32P, _I64, _U32P, _I64, _I64, _I64, _U32P, _I64, _I64P]),
    "mmm_cu_divmod": (C.c_int, [_I64, _U32P, _I64, _U32P, _I64, _I64, _U32P, _I64, _I64P, _U32P,
                                _I64, _I64P]),
    "mmm_cu_divmod_fast": (C.c_int, [_I64, _U32P, _I64, _U32P, _I64, _U32P, _I64, _I64P, _U32P,
                                     _I64, _I64P]),
    "mmm_cu_divmod_fast_dev": (C.c_int, [_I64, _VP, _I64, _VP, _I64, _VP, _VP, _VP]),
    "mmm_cu_ntt_shape": (C.c_int, [_I64, _I64, _I64P, _I64P]),
    "mmm_cu_ntt_phase_dev": (C.c_int, [_I64, C.c_int, _VP, _I64, _VP, _I64, _I64, _I64, _VP, _VP,
                                       _VP, _VP]),
    "mmm_cu_gcd": (C.c_int, [_I64, _U32P, _I64, _U32P, _I64, _I64, _U32P, _I64, _I64P]),
    "mmm_cu_ntt_mul": (C.c_int, [_I64, _U32P, _I64, _U32P, _I64, _U32P, _I64, _I64P]),
    "mmm_cu_mul_batched": (C.c_int, [_I64, _U32P, _I64, _I64, _U32P, _I64, _I64, _I64, _I64,
                                     _U32P, _I64]),
    "mmm_cu_divmod_batched": (C.c_int, [_I64, _U32P, _I64, _I64, _U32P, _I64, _I64, _I64, _I64,
                                        _U32P, _I64, _U32P, _I64]),
    "mmm_cu_ntt_mul_batched": (C.c_int, [_I64, _U32P, _I64, _I64, _U32P, _I64, _I64, _I64, _U32P,
                                         _I64]),
    "mmm_cu_mul_dev": (C.c_int, [_I64, _VP, _I64, _VP, _I64, _I64, _VP, _VP]),
    "mmm_cu_mul_range_dev": (C.c_int, [_I64, _VP, _I64, _VP, _I64, _I64, _I64, _I64, _VP, _VP]),
    "mmm_cu_divmod_dev": (C.c_int, [_I64, _VP, _I64, _VP, _I64, _I64, _VP, _VP, _VP]),
    "mmm_cu_gcd_dev": (C.c_int, [_I64, _VP, _I64, _VP, _I64, _I64, _VP, _VP, _VP]),
    "mmm_cu_ntt_mul_dev": (C.c_int, [_I64, _VP, _I64, _VP, _I64, _VP, _VP]),
    "mmm_cu_mul_batched_dev": (C.c_int, [_I64, _VP, _I64, _I64, _VP, _I64, _I64, _I64, _I64, _VP,
                                         _I64, _VP]),
    "mmm_cu_divmod_batched_dev": (C.c_int, [_I64, _VP, _I64, _I64, _VP, _I64, _I64, _I64, _I64,
                                            _VP, _I64, _VP, _I64, _VP]),
    "mmm_cu_ntt_mul_batched_dev": (C.c_int, [_I64, _VP, _I64, _I64, _VP, _I64, _I64, _I64, _VP,
                                             _I64, _VP]),
    "mmm_cu_fanout_copy_dev": (C.c_int, [_VP, _I64, C.POINTER(C.c_void_p), C.c_int32, _VP]),
    "mmm_cu_mul_range_fanout_dev": (C.c_int, [_I64, _VP, _I64, _VP, _I64, _I64, _I64, _I64,
                                              C.POINTER(C.c_void_p), C.c_int32, _VP]),
    "mmm_cu_mul_batched_fanout_dev": (C.c_int, [_I64, _VP, _I64, _I64, _VP, _I64, _I64, _I64,
                                                _I64, C.POINTER(C.c_void_p), C.c_int32, _I64,
                                                _VP]),
    "mmm_cu_divmod_batched_fanout_dev": (C.c_int, [_I64, _VP, _I64, _I64, _VP, _I64, _I64, _I64,
                                                   _I64, C.POINTER(C.c_void_p), _I64,
                                                   C.POINTER(C.c_void_p), _I64, C.c_int32, _VP]),
    "mmm_cu_mul_batched_multi": (C.c_int, [_I64, _U32P, _I64, _I64, _U32P, _I64, _I64, _I64, _I64,
                                           _U32P, _I64, _I32P, C.c_int32]),
    "mmm_cu_divmod_batched_multi": (C.c_int, [_I64, _U32P, _I64, _I64, _U32P, _I64, _I64, _I64,
                                              _I64, _U32P, _I64, _U32P, _I64, _I32P, C.c_int32]),
    "mmm_cu_ntt_mul_batched_multi": (C.c_int, [_I64, _U32P, _I64, _I64, _U32P, _I64, _I64, _I64,
                                               _U32P, _I64, _I32P, C.c_int32]),
    "mmm_cu_mul_batched_multi_dev": (C.c_int, [_I64, _VP, _I64, _I64, _VP, _I64, _I64, _I64, _I64,
                                               _VP, _I64, _I32P, C.c_int32, _VP]),
    "mmm_cu_divmod_batched_multi_dev": (C.c_int, [_I64, _VP, _I64, _I64, _VP, _I64, _I64, _I64,
                                                  _I64, _VP, _I64, _VP, _I64, _I32P, C.c_int32,
                                                  _VP]),
    "mmm_cu_ntt_mul_batched_multi_dev": (C.c_int, [_I64, _VP, _I64, _I64, _VP, _I64, _I64, _I64,
                                                   _VP, _I64, _I32P, C.c_int32, _VP]),
}

_lib: Optional[C.CDLL] = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load (once) and bind the CUDA library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run __graft_entry__.build() "
                          "(make -C paper_1402_0264_b200/csrc)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(status: int) -> None:
    if status:
        msg = load().mmm_last_error().decode(errors="replace")
        raise _ERR.get(status, MmmError)(msg)


def _u32(x) -> np.ndarray:
    a = np.asarray(x)
    if a.dtype != np.uint32:
        if a.size and (a.min() < 0 or a.max() > 0xFFFFFFFF):
            raise InvalidArgument("coefficients must be canonical field elements")
        a = a.astype(np.uint32)
    return np.ascontiguousarray(a.reshape(-1) if a.ndim <= 1 else a)


def _p(a: np.ndarray):
    return a.ctypes.data_as(_U32P)


def launch_count() -> int:
    return int(load().mmm_cu_launch_count())


class Field:
    """Prime field Z/pZ (mirrors mmm::Field, field.hpp:9-39)."""

    def __init__(self, p: int):
        _check(load().mmm_field_check(int(p)))
        self._p = int(p)

    def p(self) -> int:
        return self._p

    def add(self, a, b):
        s = a + b
        return s - self._p if s >= self._p else s

    def sub(self, a, b):
        s = a - b
        return s + self._p if s < 0 else s

    def mul(self, a, b):
        return (a * b) % self._p

    def neg(self, a):
        return 0 if a == 0 else self._p - a

    def inv(self, a) -> int:
        out = C.c_int64(0)
        _check(load().mmm_field_inv(int(a), self._p, C.byref(out)))
        return out.value

    def divide(self, a, b):
        return self.mul(a, self.inv(b))

    def reduce(self, x):
        return x % self._p


class Rng:
    """std::mt19937_64 (the reference's input generator engine)."""

    def __init__(self, seed: int):
        self._h = load().mmm_rng_create(C.c_uint64(seed & (2**64 - 1)))
        if not self._h:
            raise MemoryError("mmm_rng_create")

    def __call__(self) -> int:
        return int(load().mmm_rng_next(self._h))

    next = __call__

    def random_poly(self, terms: int, p: int) -> np.ndarray:
        out = np.zeros(max(int(terms), 1), dtype=np.uint32)
        _check(load().mmm_random_poly(self._h, int(terms), int(p), _p(out)))
        return out

    def __del__(self):
        try:
            if self._h and _lib is not None:
                _lib.mmm_rng_destroy(self._h)
        except Exception:
            pass


def random_poly(rng: Rng, terms: int, F) -> np.ndarray:
    """random_poly (poly.cpp:20-29)."""
    return rng.random_poly(terms, F.p() if isinstance(F, Field) else int(F))


def _out(out, shape):
    """A caller-supplied result array (e.g. pinned host memory, so the
    device-to-host copy runs at full link speed) or a new one."""
    if out is None:
        return np.zeros(shape, dtype=np.uint32)
    if out.dtype != np.uint32 or not out.flags.c_contiguous or tuple(out.shape) != tuple(shape):
        raise InvalidArgument(f"out: need a C-contiguous uint32 array of shape {tuple(shape)}")
    return out


def _host_free(ptr: int) -> None:
    try:
        if _lib is not None:
            _lib.mmm_cu_host_free(C.c_void_p(ptr))
    except Exception:  # interpreter teardown
        pass


def _pinned_out(out, shape):
    """A batched call's results: the caller's array, or page-locked memory from
    the library's pool (mmm_cu_host_alloc), so the device-to-host copies run at
    link speed; the buffer goes back to the pool when the array and every view
    of it are gone.  Every word is written by the call."""
    if out is not None:
        return _out(out, shape)
    n = int(np.prod(shape))
    ptr = C.c_void_p()
    _check(load().mmm_cu_host_alloc(max(n, 1) * 4, C.byref(ptr)))
    buf = (C.c_uint32 * max(n, 1)).from_address(ptr.value)
    weakref.finalize(buf, _host_free, ptr.value)
    return np.frombuffer(buf, dtype=np.uint32, count=n).reshape(shape)


def _pint(p) -> int:
    return p.p() if isinstance(p, Field) else int(p)


# ------------------------------------------------------------- host API ---
def mul(a, b, p, s: int = 0, l: int = 128, out=None) -> np.ndarray:
    a, b, p = _u32(a), _u32(b), _pint(p)
    f = _out(out, (max(a.size + b.size - 1, 1),))
    n = C.c_int64(0)
    _check(load().mmm_cu_mul(p, _p(a), a.size, _p(b), b.size, s, l, _p(f), f.size, C.byref(n)))
    return f[: n.value] if out is not None else f[: n.value].copy()


def divmod(a, b, p, s: int = 64):
    a, b, p = _u32(a), _u32(b), _pint(p)
    q = np.zeros(max(a.size, 1), dtype=np.uint32)
    r = np.zeros(max(a.size, b.size, 1), dtype=np.uint32)
    nq, nr = C.c_int64(0), C.c_int64(0)
    _check(load().mmm_cu_divmod(p, _p(a), a.size, _p(b), b.size, s, _p(q), q.size, C.byref(nq),
                                _p(r), r.size, C.byref(nr)))
    return q[: nq.value].copy(), r[: nr.value].copy()


def divmod_fast(a, b, p):
    """divmod(a, b) by Newton iteration and NTT products: the same (q, r)."""
    a, b, p = _u32(a), _u32(b), _pint(p)
    q = np.zeros(max(a.size, 1), dtype=np.uint32)
    r = np.zeros(max(a.size, b.size, 1), dtype=np.uint32)
    nq, nr = C.c_int64(0), C.c_int64(0)
    _check(load().mmm_cu_divmod_fast(p, _p(a), a.size, _p(b), b.size, _p(q), q.size, C.byref(nq),
                                     _p(r), r.size, C.byref(nr)))
    return q[: nq.value].copy(), r[: nr.value].copy()


def divmod_fast_dev(p, d_a, na, d_b, nb, d_q, d_r, stream=0):
    _check(load().mmm_cu_divmod_fast_dev(_pint(p), d_a, na, d_b, nb, d_q, d_r, stream))


def ntt_shape(p, nf):
    """(n1, n2): the four-step split of the NTT for an nf-word product."""
    n1, n2 = C.c_int64(0), C.c_int64(0)
    _check(load().mmm_cu_ntt_shape(_pint(p), nf, C.byref(n1), C.byref(n2)))
    return n1.value, n2.value


def ntt_phase_dev(p, phase, d_a, na, d_b, nb, start, n, d_work_a, d_work_b, d_f, stream=0):
    """One phase of the sharded four-step NTT product (see include/mmm_cu.h)."""
    _check(load().mmm_cu_ntt_phase_dev(_pint(p), phase, d_a, na, d_b, nb, start, n, d_work_a,
                                       d_work_b, d_f, stream))


def gcd(a, b, p, s: int = 64) -> np.ndarray:
    a, b, p = _u32(a), _u32(b), _pint(p)
    g = np.zeros(max(a.size, b.size, 1), dtype=np.uint32)
    n = C.c_int64(0)
    _check(load().mmm_cu_gcd(p, _p(a), a.size, _p(b), b.size, s, _p(g), g.size, C.byref(n)))
    return g[: n.value].copy()


def ntt_mul(a, b, p, out=None) -> np.ndarray:
    a, b, p = _u32(a), _u32(b), _pint(p)
    f = _out(out, (max(a.size + b.size - 1, 1),))
    n = C.c_int64(0)
    _check(load().mmm_cu_ntt_mul(p, _p(a), a.size, _p(b), b.size, _p(f), f.size, C.byref(n)))
    return f[: n.value] if out is not None else f[: n.value].copy()


def mul_batched(A, B, p, s: int = 0, out=None) -> np.ndarray:
    A, B, p = _u32(A), _u32(B), _pint(p)
    cnt, na = A.shape
    nb = B.shape[1]
    F = _pinned_out(out, (cnt, na + nb - 1))
    _check(load().mmm_cu_mul_batched(p, _p(A), na, na, _p(B), nb, nb, cnt, s, _p(F), F.shape[1]))
    return F


def divmod_batched(A, B, p, s: int = 0, q_out=None, r_out=None):
    A, B, p = _u32(A), _u32(B), _pint(p)
    cnt, na = A.shape
    nb = B.shape[1]
    Q = _pinned_out(q_out, (cnt, na - nb + 1))
    R = _pinned_out(r_out, (cnt, max(nb - 1, 1)))
    _check(load().mmm_cu_divmod_batched(p, _p(A), na, na, _p(B), nb, nb, cnt, s, _p(Q),
                                        Q.shape[1], _p(R), R.shape[1]))
    return Q, R[:, : nb - 1]


def ntt_mul_batched(A, B, p, out=None) -> np.ndarray:
    A, B, p = _u32(A), _u32(B), _pint(p)
    cnt, na = A.shape
    nb = B.shape[1]
    F = _pinned_out(out, (cnt, na + nb - 1))
    _check(load().mmm_cu_ntt_mul_batched(p, _p(A), na, na, _p(B), nb, nb, cnt, _p(F),
                                         F.shape[1]))
    return F


# -------------------------------------------- device-pointer API (async) --
# Pointers are integers (e.g. torch.Tensor.data_ptr()), stream a
# cudaStream_t as int (torch.cuda.Stream.cuda_stream) or 0.
def mul_dev(p, d_a, na, d_b, nb, d_f, s=0, stream=0):
    _check(load().mmm_cu_mul_dev(_pint(p), d_a, na, d_b, nb, s, d_f, stream))


def mul_range_dev(p, d_a, na, d_b, nb, k0, k1, d_f, s=0, stream=0):
    """Product coefficients [k0, k1) into d_f[0, k1 - k0) (a rank's output slice)."""
    _check(load().mmm_cu_mul_range_dev(_pint(p), d_a, na, d_b, nb, k0, k1, s, d_f, stream))


def divmod_dev(p, d_a, na, d_b, nb, d_q, d_r, s=64, stream=0):
    _check(load().mmm_cu_divmod_dev(_pint(p), d_a, na, d_b, nb, s, d_q, d_r, stream))


def gcd_dev(p, d_a, na, d_b, nb, d_g, d_ng, s=64, stream=0):
    _check(load().mmm_cu_gcd_dev(_pint(p), d_a, na, d_b, nb, s, d_g, d_ng, stream))


def ntt_mul_dev(p, d_a, na, d_b, nb, d_f, stream=0):
    _check(load().mmm_cu_ntt_mul_dev(_pint(p), d_a, na, d_b, nb, d_f, stream))


def mul_batched_dev(p, d_A, lda, na, d_B, ldb, nb, count, d_F, ldf, s=0, stream=0):
    _check(load().mmm_cu_mul_batched_dev(_pint(p), d_A, lda, na, d_B, ldb, nb, count, s, d_F,
                                         ldf, stream))


def divmod_batched_dev(p, d_A, lda, na, d_B, ldb, nb, count, d_Q, ldq, d_R, ldr, s=0,
                       stream=0):
    _check(load().mmm_cu_divmod_batched_dev(_pint(p), d_A, lda, na, d_B, ldb, nb, count, s, d_Q,
                                            ldq, d_R, ldr, stream))


def ntt_mul_batched_dev(p, d_A, lda, na, d_B, ldb, nb, count, d_F, ldf, stream=0):
    _check(load().mmm_cu_ntt_mul_batched_dev(_pint(p), d_A, lda, na, d_B, ldb, nb, count, d_F,
                                             ldf, stream))


# ------------------------------------------------- fan-out (fused gather) --
# `outs` lists device pointers (ints) with one layout; each output word is
# stored into every one of them -- with every rank's buffer (symmetric memory
# over NVLink) the gather of a sharded batch happens in the kernel's epilogue.
def _ptrs(outs):
    outs = [int(x) for x in outs]
    return (C.c_void_p * len(outs))(*outs), len(outs)


def mul_range_fanout_dev(p, d_a, na, d_b, nb, k0, k1, outs, s=8, stream=0):
    arr, n = _ptrs(outs)
    _check(load().mmm_cu_mul_range_fanout_dev(_pint(p), d_a, na, d_b, nb, k0, k1, s, arr, n,
                                              stream))


def mul_batched_fanout_dev(p, d_A, lda, na, d_B, ldb, nb, count, outs, ldf, s=0, stream=0):
    arr, n = _ptrs(outs)
    _check(load().mmm_cu_mul_batched_fanout_dev(_pint(p), d_A, lda, na, d_B, ldb, nb, count, s,
                                                arr, n, ldf, stream))


def divmod_batched_fanout_dev(p, d_A, lda, na, d_B, ldb, nb, count, q_outs, ldq, r_outs, ldr,
                              s=0, stream=0):
    if len(q_outs) != len(r_outs):
        raise InvalidArgument("division batch: q and r fan-outs differ in length")
    qa, n = _ptrs(q_outs)
    ra, _ = _ptrs(r_outs)
    _check(load().mmm_cu_divmod_batched_fanout_dev(_pint(p), d_A, lda, na, d_B, ldb, nb, count, s,
                                                   qa, ldq, ra, ldr, n, stream))


def fanout_copy_dev(d_src, n, outs, stream=0):
    """n words of d_src into every device buffer of `outs` (one peer-store kernel)."""
    arr, k = _ptrs(outs)
    _check(load().mmm_cu_fanout_copy_dev(d_src, n, arr, k, stream))


# ------------------------------------------ several GPUs from one process --
# `devices`: device ordinals (repeats allowed); the batch splits into
# contiguous shares, one per entry (include/mmm_cu.h, "several GPUs").
def _devs(devices):
    d = np.ascontiguousarray(np.asarray(list(devices), dtype=np.int32))
    return d.ctypes.data_as(_I32P), d.size, d


def mul_batched_multi(A, B, p, devices, s: int = 0, out=None) -> np.ndarray:
    A, B, p = _u32(A), _u32(B), _pint(p)
    cnt, na = A.shape
    nb = B.shape[1]
    F = _out(out, (cnt, na + nb - 1))
    dp, nd, _keep = _devs(devices)
    _check(load().mmm_cu_mul_batched_multi(p, _p(A), na, na, _p(B), nb, nb, cnt, s, _p(F),
                                           F.shape[1], dp, nd))
    return F


def divmod_batched_multi(A, B, p, devices, s: int = 0):
    A, B, p = _u32(A), _u32(B), _pint(p)
    cnt, na = A.shape
    nb = B.shape[1]
    Q = np.zeros((cnt, na - nb + 1), dtype=np.uint32)
    R = np.zeros((cnt, max(nb - 1, 1)), dtype=np.uint32)
    dp, nd, _keep = _devs(devices)
    _check(load().mmm_cu_divmod_batched_multi(p, _p(A), na, na, _p(B), nb, nb, cnt, s, _p(Q),
                                              Q.shape[1], _p(R), R.shape[1], dp, nd))
    return Q, R[:, : nb - 1]


def ntt_mul_batched_multi(A, B, p, devices, out=None) -> np.ndarray:
    A, B, p = _u32(A), _u32(B), _pint(p)
    cnt, na = A.shape
    nb = B.shape[1]
    F = _out(out, (cnt, na + nb - 1))
    dp, nd, _keep = _devs(devices)
    _check(load().mmm_cu_ntt_mul_batched_multi(p, _p(A), na, na, _p(B), nb, nb, cnt, _p(F),
                                               F.shape[1], dp, nd))
    return F


def mul_batched_multi_dev(p, d_A, lda, na, d_B, ldb, nb, count, d_F, ldf, devices, s=0,
                          stream=0):
    dp, nd, _keep = _devs(devices)
    _check(load().mmm_cu_mul_batched_multi_dev(_pint(p), d_A, lda, na, d_B, ldb, nb, count, s,
                                               d_F, ldf, dp, nd, stream))


def divmod_batched_multi_dev(p, d_A, lda, na, d_B, ldb, nb, count, d_Q, ldq, d_R, ldr, devices,
                             s=0, stream=0):
    dp, nd, _keep = _devs(devices)
    _check(load().mmm_cu_divmod_batched_multi_dev(_pint(p), d_A, lda, na, d_B, ldb, nb, count, s,
                                                  d_Q, ldq, d_R, ldr, dp, nd, stream))


def ntt_mul_batched_multi_dev(p, d_A, lda, na, d_B, ldb, nb, count, d_F, ldf, devices, stream=0):
    dp, nd, _keep = _devs(devices)
    _check(load().mmm_cu_ntt_mul_batched_multi_dev(_pint(p), d_A, lda, na, d_B, ldb, nb, count,
                                                   d_F, ldf, dp, nd, stream))


def release_scratch() -> None:
    """Free this thread's streams, arenas and staging (mmm_cu_release_scratch)."""
    _check(load().mmm_cu_release_scratch())


def last_schedule():
    """[(name, blocks, threads)] of the kernels this thread's last host call launched."""
    n = C.c_int32(0)
    _check(load().mmm_cu_last_schedule(None, 0, C.byref(n)))
    recs = (KernelRec * max(n.value, 1))()
    _check(load().mmm_cu_last_schedule(recs, n.value, C.byref(n)))
    return [(r.name.decode(), r.blocks, r.threads) for r in recs[: n.value]]
