#!/usr/bin/env python3
"""Generate tests/golden/*.json from the REFERENCE ITSELF (oracle/_ref).

Run in the build container, where /root/reference exists and
``make -C oracle`` has compiled the unmodified reference oracle into
oracle/_ref/libref_oracle.so:

    python tests/golden/make_golden.py            # golden_small.json (seconds)
    python tests/golden/make_golden.py --scale    # golden_configs.json (minutes, all cores)

Inputs are drawn with the reference's own std::mt19937_64 + random_poly (via
ref_shim.cpp), in the draw order of each reference test (see suites.py).
Outputs are recorded as digests: sha256 of the trimmed coefficient array as
little-endian int64, first 16 hex digits ("" for the zero polynomial).
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from oracle import pyoracle  # noqa: E402
import suites  # noqa: E402


def digest(x) -> str:
    a = np.ascontiguousarray(np.asarray(x, dtype="<i8"))
    return hashlib.sha256(a.tobytes()).hexdigest()[:16] if a.size else ""


class RefRng:
    """The reference's std::mt19937_64 and random_poly behind ref_shim.cpp."""

    def __init__(self, ref: pyoracle.Reference, seed: int):
        self.ref, self.h = ref, ref.rng_new(seed)

    def next(self) -> int:
        return self.ref.rng_next(self.h)

    def random_poly(self, terms: int, p: int) -> np.ndarray:
        out = np.zeros(terms, dtype=np.int64)
        st = self.ref._random_poly(self.h, terms, p, out.ctypes.data_as(C.POINTER(C.c_int64)))
        assert st == 0
        return out

    def __del__(self):
        try:
            self.ref.rng_free(self.h)
        except Exception:
            pass


def record(ref, case: dict) -> dict:
    p, a, b = case["p"], case["a"], case["b"]
    out = {k: v for k, v in case.items() if k not in ("a", "b", "am", "g")}
    out["a"], out["b"] = digest(a), digest(b)
    out["na"], out["nb"] = int(len(a)), int(len(b))
    op = case["op"]
    if op in ("mul", "all"):
        out["f"] = digest(ref.mul(a, b, p))
    if op in ("divmod", "all", "verify"):
        q, r = ref.divmod(a, b, p)
        out["q"], out["r"] = digest(q), digest(r)
    if op in ("gcd", "all", "verify"):
        out["g"] = digest(ref.gcd(a, b, p))
    if op == "verify":
        out["am"] = digest(case["am"])
        out["f"] = digest(ref.mul(case["am"], b, p))
    return out


def make_small(ref) -> dict:
    mul = ref.mul
    res = {"digest": "sha256(trimmed coeffs as <i8)[:16]", "suites": {}}
    plans = [
        ("mutual_oracle", 2026, suites.mutual_oracle),
        ("divmod_roundtrip", 123, suites.divmod_roundtrip),
        ("planted_gcd", 5150, suites.planted_gcd),
        ("division_sweep", 424242, suites.division_sweep),
        ("multiplication_sweep", 1337, suites.multiplication_sweep),
        ("gcd_sweep", 4242, suites.gcd_sweep),
    ]
    for name, seed, gen in plans:
        rng = RefRng(ref, seed)
        res["suites"][name] = {"seed": seed, "cases": [record(ref, c) for c in gen(rng, mul)]}
    res["suites"]["acceptance"] = {
        "seed": "20260819+p",
        "cases": [record(ref, c) for c in suites.acceptance(lambda s: RefRng(ref, s), mul)],
    }
    for p in (7, 101, suites.P_BENCH):
        rng = RefRng(ref, 42)
        res["suites"][f"verify_p{p}"] = {
            "seed": 42, "cases": [record(ref, c) for c in suites.verify(rng, p)]}
    frozen = []
    for c in suites.FROZEN:
        p = c["p"]
        a = suites.materialise(c["a"], p, mul)
        b = suites.materialise(c["b"], p, mul)
        e = {"op": c["op"], "p": p, "a": a.tolist(), "b": b.tolist()}
        if c["op"] == "mul":
            e["f"] = ref.mul(a, b, p).tolist()
            assert c["f"] is None or e["f"] == c["f"], (c, e)
        elif c["op"] == "divmod":
            q, r = ref.divmod(a, b, p)
            e["q"], e["r"] = q.tolist(), r.tolist()
            assert c["q"] is None or (e["q"] == c["q"] and e["r"] == c["r"]), (c, e)
        else:
            e["g"] = ref.gcd(a, b, p).tolist()
            assert c["g"] is None or e["g"] == c["g"], (c, e)
        frozen.append(e)
    res["frozen"] = frozen
    return res


def _par_mul_alt(port: pyoracle.Port, a, b, p, threads):
    """One large product split over output ranges (oracle_mul_alt restated)."""
    nf = len(a) + len(b) - 1
    out = np.zeros(nf, dtype=np.int64)
    fn = port.lib.orc_poly_mul_alt_range
    P = C.POINTER(C.c_int64)
    fn.argtypes = [P, C.c_int64, P, C.c_int64, C.c_int64, C.c_int64, C.c_int64, P]
    fn.restype = None
    # balance the triangular work profile: equal-work output cuts
    w = np.minimum(np.arange(nf) + 1, nf - np.arange(nf)).astype(np.float64)
    cuts = np.searchsorted(np.cumsum(w), np.linspace(0, w.sum(), 8 * threads + 1)[1:-1])
    bounds = [0, *cuts.tolist(), nf]
    ap, bp_ = a.ctypes.data_as(P), b.ctypes.data_as(P)

    def run(i):
        k0, k1 = bounds[i], bounds[i + 1]
        if k1 > k0:
            fn(ap, len(a), bp_, len(b), p, k0, k1,
               out[k0:].ctypes.data_as(P))

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, range(len(bounds) - 1)))
    n = int(np.flatnonzero(out)[-1]) + 1 if out.any() else 0
    return out[:n]


def make_scale(ref, threads: int, big: bool) -> dict:
    port = pyoracle.Port()
    P = suites.P_BENCH
    res = {"digest": "sha256(trimmed coeffs as <i8)[:16]", "p": P, "seed": 42}
    t0 = time.time()
    c = suites.cfg1(RefRng(ref, 42))
    res["cfg1"] = {"a": digest(c["a"]), "b": digest(c["b"]), "f": digest(ref.mul(c["a"], c["b"], P))}
    print(f"cfg1 {time.time() - t0:.1f}s", flush=True)
    c = suites.cfg2(RefRng(ref, 42), ref.mul, port.monic)
    g = ref.gcd(c["a"], c["b"], P)
    steps, updates = port.gcd_count(c["a"], c["b"], P)
    res["cfg2"] = {"a": digest(c["a"]), "b": digest(c["b"]), "g": digest(g), "deg_g": len(g) - 1,
                   "g_equals_planted": bool(np.array_equal(g, c["g"])), "steps": steps,
                   "updates": updates}
    print(f"cfg2 {time.time() - t0:.1f}s", flush=True)
    c = suites.cfg3(RefRng(ref, 42))
    q, r = ref.divmod(c["a"], c["b"], P)
    res["cfg3"] = {"a": digest(c["a"]), "b": digest(c["b"]), "q": digest(q), "r": digest(r),
                   "nq": len(q), "nr": len(r)}
    print(f"cfg3 {time.time() - t0:.1f}s", flush=True)

    rng = RefRng(ref, 42)
    c = suites.cfg4_big(rng)
    res["cfg4_big"] = {"a": digest(c["a"]), "b": digest(c["b"])}
    if big:
        f = _par_mul_alt(port, c["a"], c["b"], P, threads)
        res["cfg4_big"]["f"] = digest(f)
        print(f"cfg4 big {time.time() - t0:.1f}s", flush=True)
    cb = suites.cfg4_batch(rng)
    with ThreadPoolExecutor(threads) as ex:
        fs = list(ex.map(lambda i: digest(ref.mul(cb["A"][i], cb["B"][i], P)), range(256)))
    res["cfg4_batch"] = {"A": digest(cb["A"]), "B": digest(cb["B"]), "f": fs,
                         "f_all": hashlib.sha256("".join(fs).encode()).hexdigest()[:16]}
    print(f"cfg4 batch {time.time() - t0:.1f}s", flush=True)

    c5 = suites.cfg5(RefRng(ref, 42))
    with ThreadPoolExecutor(threads) as ex:
        fs = list(ex.map(lambda i: digest(ref.mul(c5["A"][i], c5["B"][i], P)), range(4096)))
        qr = list(ex.map(lambda i: ref.divmod(c5["C"][i], c5["D"][i], P), range(4096)))
    qs = [digest(q) for q, _ in qr]
    rs = [digest(r) for _, r in qr]
    res["cfg5"] = {"A": digest(c5["A"]), "B": digest(c5["B"]), "C": digest(c5["C"]),
                   "D": digest(c5["D"]), "f": fs, "q": qs, "r": rs,
                   "f_all": hashlib.sha256("".join(fs).encode()).hexdigest()[:16],
                   "qr_all": hashlib.sha256("".join(qs + rs).encode()).hexdigest()[:16]}
    print(f"cfg5 {time.time() - t0:.1f}s", flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", action="store_true")
    ap.add_argument("--big", action="store_true", help="include the 2^20 x 2^20 product")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    ref = pyoracle.Reference()
    if args.scale:
        out = os.path.join(HERE, "golden_configs.json")
        old = json.load(open(out)) if os.path.exists(out) else {}
        res = make_scale(ref, args.threads, args.big)
        if not args.big and "f" in old.get("cfg4_big", {}) and \
                old["cfg4_big"].get("a") == res["cfg4_big"]["a"]:
            res["cfg4_big"]["f"] = old["cfg4_big"]["f"]
    else:
        out = os.path.join(HERE, "golden_small.json")
        res = make_small(ref)
    with open(out, "w") as fh:
        json.dump(res, fh, indent=None, separators=(",", ":"))
        fh.write("\n")
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
