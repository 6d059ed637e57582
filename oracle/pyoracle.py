"""ctypes face of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two backends with one API:

* ``Port``      -- oracle/liboracle_port.so, the plain-C restatement (oracle.c);
* ``Reference`` -- oracle/_ref/libref_oracle.so, the unmodified reference
  oracle (/root/reference/proj/src/{field,poly,oracle}.cpp) behind ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) import this module, as the checker or as the timed CPU
baseline.  The product package never does.

Polynomials are numpy int64 arrays, ascending, trimmed (zero = empty array),
like mmm::Poly (proj/include/mmm/poly.hpp:16-30).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle_port.so")
REF_SO = os.path.join(HERE, "_ref", "libref_oracle.so")

_I64P = C.POINTER(C.c_int64)


class OracleError(Exception):
    pass


class InvalidArgument(OracleError, ValueError):
    pass


class DomainError(OracleError, ArithmeticError):
    pass


def _raise(status: int, what: str) -> None:
    if status == 1:
        raise InvalidArgument(what)
    if status == 2:
        raise DomainError(what)
    if status != 0:
        raise OracleError(f"{what}: status {status}")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_I64P)


def _arr(x) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.int64))
    return a if a.size else np.zeros(1, dtype=np.int64)[:0]


def build_port() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)


class _Backend:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.lib = C.CDLL(path)
        self._bind()

    def _fn(self, name, res, *args):
        f = getattr(self.lib, self.prefix + name)
        f.restype = res
        f.argtypes = list(args)
        return f

    # -- polynomial entry points shared by both backends ------------------
    def mul(self, a, b, p: int) -> np.ndarray:
        a, b = _arr(a), _arr(b)
        out = np.zeros(max(a.size + b.size - 1, 1), dtype=np.int64)
        n = self._mul(_ptr(a), a.size, _ptr(b), b.size, p, _ptr(out))
        return out[:n].copy()

    def mul_alt(self, a, b, p: int) -> np.ndarray:
        a, b = _arr(a), _arr(b)
        out = np.zeros(max(a.size + b.size - 1, 1), dtype=np.int64)
        n = self._mul_alt(_ptr(a), a.size, _ptr(b), b.size, p, _ptr(out))
        return out[:n].copy()

    def divmod(self, a, b, p: int):
        a, b = _arr(a), _arr(b)
        q = np.zeros(max(a.size, 1), dtype=np.int64)
        r = np.zeros(max(a.size, 1), dtype=np.int64)
        nq, nr = C.c_int64(0), C.c_int64(0)
        st = self._divmod(_ptr(a), a.size, _ptr(b), b.size, p, _ptr(q), C.byref(nq), _ptr(r),
                          C.byref(nr))
        _raise(st, "divmod: division by the zero polynomial")
        return q[: nq.value].copy(), r[: nr.value].copy()

    def gcd(self, a, b, p: int) -> np.ndarray:
        a, b = _arr(a), _arr(b)
        g = np.zeros(max(a.size, b.size, 1), dtype=np.int64)
        ng = C.c_int64(0)
        st = self._gcd(_ptr(a), a.size, _ptr(b), b.size, p, _ptr(g), C.byref(ng))
        _raise(st, "gcd: both inputs are zero")
        return g[: ng.value].copy()


class Port(_Backend):
    """The plain-C restatement (oracle/oracle.c)."""

    prefix = "orc_"

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build_port()
        super().__init__(path)

    def _bind(self):
        I64 = C.c_int64
        self.field_check = self._fn("field_check", C.c_int, I64)
        self.inv_raw = self._fn("inv", I64, I64, I64)
        self._mul = self._fn("poly_mul", I64, _I64P, I64, _I64P, I64, I64, _I64P)
        self._mul_alt = self._fn("poly_mul_alt", I64, _I64P, I64, _I64P, I64, I64, _I64P)
        self._add = self._fn("poly_add", I64, _I64P, I64, _I64P, I64, I64, _I64P)
        self._sub = self._fn("poly_sub", I64, _I64P, I64, _I64P, I64, I64, _I64P)
        self._monic = self._fn("monic", I64, _I64P, I64, I64, _I64P)
        self._divmod = self._fn("divmod", C.c_int, _I64P, I64, _I64P, I64, I64, _I64P, _I64P,
                                _I64P, _I64P)
        self._gcd = self._fn("gcd", C.c_int, _I64P, I64, _I64P, I64, I64, _I64P, _I64P)
        self._gcd_count = self._fn("gcd_count", C.c_int, _I64P, I64, _I64P, I64, I64, _I64P,
                                   _I64P)
        self.add_s = self._fn("add", I64, I64, I64, I64)
        self.sub_s = self._fn("sub", I64, I64, I64, I64)
        self.mul_s = self._fn("mulmod", I64, I64, I64, I64)
        self.reduce_s = self._fn("reduce", I64, I64, I64)

    def add(self, a, b, p):
        a, b = _arr(a), _arr(b)
        out = np.zeros(max(a.size, b.size, 1), dtype=np.int64)
        return out[: self._add(_ptr(a), a.size, _ptr(b), b.size, p, _ptr(out))].copy()

    def sub(self, a, b, p):
        a, b = _arr(a), _arr(b)
        out = np.zeros(max(a.size, b.size, 1), dtype=np.int64)
        return out[: self._sub(_ptr(a), a.size, _ptr(b), b.size, p, _ptr(out))].copy()

    def monic(self, a, p):
        a = _arr(a)
        out = np.zeros(max(a.size, 1), dtype=np.int64)
        return out[: self._monic(_ptr(a), a.size, p, _ptr(out))].copy()

    def inv(self, a: int, p: int) -> int:
        r = self.inv_raw(a, p)
        if r < 0:
            raise DomainError("field: inverse of zero")
        return r

    def gcd_count(self, a, b, p):
        """(head eliminations, coefficient updates) of the Euclid run."""
        a, b = _arr(a), _arr(b)
        s, u = C.c_int64(0), C.c_int64(0)
        _raise(self._gcd_count(_ptr(a), a.size, _ptr(b), b.size, p, C.byref(s), C.byref(u)),
               "gcd")
        return s.value, u.value


class Reference(_Backend):
    """The unmodified reference oracle compiled into oracle/_ref/."""

    prefix = "ref_"

    def __init__(self, path: str = REF_SO):
        super().__init__(path)

    def _bind(self):
        I64 = C.c_int64
        self.field_check = self._fn("field_check", C.c_int, I64)
        self.inv_raw = self._fn("inv", I64, I64, I64)
        self.rng_new = self._fn("rng_new", C.c_void_p, C.c_uint64)
        self.rng_free = self._fn("rng_free", None, C.c_void_p)
        self.rng_next = self._fn("rng_next", C.c_uint64, C.c_void_p)
        self._random_poly = self._fn("random_poly", C.c_int, C.c_void_p, I64, I64, _I64P)
        self._mul = self._fn("mul", I64, _I64P, I64, _I64P, I64, I64, _I64P)
        self._mul_alt = self._fn("mul_alt", I64, _I64P, I64, _I64P, I64, I64, _I64P)
        self._divmod = self._fn("divmod", C.c_int, _I64P, I64, _I64P, I64, I64, _I64P, _I64P,
                                _I64P, _I64P)
        self._gcd = self._fn("gcd", C.c_int, _I64P, I64, _I64P, I64, I64, _I64P, _I64P)


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def best() -> _Backend:
    """The reference build when present (kind "reference"), else the port."""
    return Reference() if reference_available() else Port()


class MT64:
    """std::mt19937_64 + libstdc++ uniform_int_distribution, restated in Python
    (mirrors oracle.c; used to pin both the C port and the product generator)."""

    N, M = 312, 156
    MASK = (1 << 64) - 1

    def __init__(self, seed: int):
        mt = [seed & self.MASK]
        for i in range(1, self.N):
            mt.append((6364136223846793005 * (mt[-1] ^ (mt[-1] >> 62)) + i) & self.MASK)
        self.mt, self.idx = mt, self.N

    def _twist(self):
        mt = self.mt
        for i in range(self.N):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % self.N] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + self.M) % self.N] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self.N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000 & self.MASK
        y ^= (y << 37) & 0xFFF7EEE000000000 & self.MASK
        y ^= y >> 43
        return y & self.MASK

    def uniform(self, lo: int, hi: int) -> int:
        erange = hi - lo + 1
        prod = self() * erange
        low = prod & self.MASK
        if low < erange:
            thr = ((1 << 64) - erange) % erange
            while low < thr:
                prod = self() * erange
                low = prod & self.MASK
        return (prod >> 64) + lo

    def random_poly(self, terms: int, p: int) -> np.ndarray:
        out = [self.uniform(0, p - 1) for _ in range(terms - 1)]
        out.append(self.uniform(1, p - 1))
        return np.array(out, dtype=np.int64)
