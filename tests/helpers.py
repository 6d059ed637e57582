"""Test helpers: digests, RNG adapters and suite replay (see golden/suites.py)."""
from __future__ import annotations

import hashlib

import numpy as np

import suites  # tests/golden on sys.path (conftest)


def digest(x) -> str:
    """sha256 of the trimmed coefficients as little-endian int64, 16 hex digits."""
    a = np.ascontiguousarray(np.asarray(x).astype("<i8"))
    return hashlib.sha256(a.tobytes()).hexdigest()[:16] if a.size else ""


class PyRng:
    """The Python restatement of mt19937_64 + random_poly (oracle/pyoracle.py)."""

    def __init__(self, seed):
        from oracle.pyoracle import MT64
        self.g = MT64(seed)

    def next(self):
        return self.g()

    def random_poly(self, terms, p):
        return self.g.random_poly(terms, p)


class PortRng:
    """The C restatement (oracle.c) -- fast, for config-scale inputs."""

    def __init__(self, port, seed):
        import ctypes as C
        self.port, self.C = port, C
        lib = port.lib
        lib.orc_mt_seed.argtypes = [C.c_void_p, C.c_uint64]
        lib.orc_mt_next.argtypes = [C.c_void_p]
        lib.orc_mt_next.restype = C.c_uint64
        lib.orc_random_poly.argtypes = [C.c_void_p, C.c_int64, C.c_int64,
                                        C.POINTER(C.c_int64)]
        self.state = C.create_string_buffer(312 * 8 + 64)
        lib.orc_mt_seed(self.state, seed)

    def next(self):
        return self.port.lib.orc_mt_next(self.state)

    def random_poly(self, terms, p):
        out = np.zeros(terms, dtype=np.int64)
        st = self.port.lib.orc_random_poly(self.state, terms, p,
                                           out.ctypes.data_as(self.C.POINTER(self.C.c_int64)))
        assert st == 0
        return out


class ProductRng:
    """The product's host generator (mmm_rng_*, std::mt19937_64 in libmmm_cu)."""

    def __init__(self, seed):
        import paper_1402_0264_b200 as mmm
        self.g = mmm.Rng(seed)

    def next(self):
        return self.g()

    def random_poly(self, terms, p):
        return self.g.random_poly(terms, p).astype(np.int64)


SEEDED = {
    "mutual_oracle": (2026, suites.mutual_oracle),
    "divmod_roundtrip": (123, suites.divmod_roundtrip),
    "planted_gcd": (5150, suites.planted_gcd),
    "division_sweep": (424242, suites.division_sweep),
    "multiplication_sweep": (1337, suites.multiplication_sweep),
    "gcd_sweep": (4242, suites.gcd_sweep),
}


def replay(name, rng_cls, mul):
    """Yield the cases of golden suite `name` with inputs drawn by rng_cls."""
    if name in SEEDED:
        seed, gen = SEEDED[name]
        yield from gen(rng_cls(seed), mul)
    elif name == "acceptance":
        yield from suites.acceptance(rng_cls, mul)
    elif name.startswith("verify_p"):
        yield from suites.verify(rng_cls(42), int(name[len("verify_p"):]))
    else:
        raise KeyError(name)
