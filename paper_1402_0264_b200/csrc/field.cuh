// field.cuh -- Z/pZ arithmetic on 32-bit canonical residues for sm_100a.
//
// Semantics follow mmm::Field (proj/include/mmm/field.hpp:9-39): elements are
// canonical residues in [0, p) of a prime p < 2^31.  The reference multiplies
// with `(a*b) % p` on int64 (field.hpp:23); here every hot-loop product is one
// IMAD.WIDE.U32 into a 64-bit accumulator, and reduction happens lazily:
//
//   fold(x)   = hi(x) * (2^32 mod p) + lo(x)        one IMAD.WIDE.U32, < p*2^32
//   redc(t)   = t * 2^-32 mod p   (Montgomery, odd p, t < p*2^32)
//   reduce(x) = x mod p = redc(redc(fold(x)) * R2)  exact for any 64-bit x
//
// p = 2 (the only even prime the reference Field accepts, test_field.cpp:12)
// has no Montgomery form; it takes a plain `%` path chosen by a warp-uniform
// branch.  Results are canonical residues, bit-identical to the reference.
#pragma once
#include <cstdint>

namespace mmm_cu {

struct FieldParams {
    uint32_t p;      // modulus, prime, 2 <= p < 2^31
    uint32_t pinv;   // p^-1 mod 2^32 (odd p)
    uint32_t r2;     // 2^64 mod p
    uint32_t c32;    // 2^32 mod p
    uint32_t odd;    // p odd -> Montgomery path
    uint32_t fold_terms;  // products (< (p-1)^2) that may be added to a folded accumulator
};

// Host-side construction.
inline FieldParams make_field(uint32_t p) {
    FieldParams F{};
    F.p = p;
    F.odd = p & 1u;
    uint32_t inv = 1;
    if (F.odd) {
        inv = p;  // Newton iteration for p^-1 mod 2^32 (p*p == 1 mod 8)
        for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
    }
    F.pinv = inv;
    uint64_t c32 = (uint64_t(1) << 32) % p;
    F.c32 = uint32_t(c32);
    F.r2 = uint32_t((c32 * c32) % p);
    // largest t with fold_max + t*(p-1)^2 < 2^64, fold_max = (2^32-1)*p
    unsigned __int128 pm1sq = (unsigned __int128)(p - 1) * (p - 1);
    unsigned __int128 head = ((unsigned __int128)1 << 64) - 1 - (unsigned __int128)0xFFFFFFFFu * p;
    unsigned __int128 t = pm1sq ? head / pm1sq : 0xFFFFFFFFu;
    F.fold_terms = t > 0x7FFFFFFF ? 0x7FFFFFFF : uint32_t(t);
    return F;
}

__device__ __forceinline__ uint64_t mad_wide(uint32_t a, uint32_t b, uint64_t c) {
    return c + uint64_t(a) * b;  // IMAD.WIDE.U32 with 64-bit addend
}

__device__ __forceinline__ uint64_t fold(uint64_t x, const FieldParams& F) {
    return mad_wide(uint32_t(x >> 32), F.c32, uint64_t(uint32_t(x)));
}

// Montgomery reduction, odd p, t < p * 2^32: returns t * 2^-32 mod p in [0, p).
__device__ __forceinline__ uint32_t redc(uint64_t t, const FieldParams& F) {
    uint32_t m = uint32_t(t) * F.pinv;
    uint32_t hi = uint32_t(t >> 32);
    uint32_t mp = __umulhi(m, F.p);
    uint32_t r = hi - mp;
    return hi < mp ? r + F.p : r;
}

// Exact x mod p for any 64-bit x.
__device__ __forceinline__ uint32_t reduce(uint64_t x, const FieldParams& F) {
    if (!F.odd) return uint32_t(x % F.p);
    uint32_t y = redc(fold(x, F), F);
    return redc(uint64_t(y) * F.r2, F);
}

// reduce() for odd p known at compile time of the caller (no p = 2 branch)
__device__ __forceinline__ uint32_t reduce_odd(uint64_t x, const FieldParams& F) {
    uint32_t y = redc(fold(x, F), F);
    return redc(uint64_t(y) * F.r2, F);
}
template <bool ODD>
__device__ __forceinline__ uint32_t reduce_t(uint64_t x, const FieldParams& F) {
    return ODD ? reduce_odd(x, F) : reduce(x, F);
}

__device__ __forceinline__ uint32_t mulmod(uint32_t a, uint32_t b, const FieldParams& F) {
    return reduce(uint64_t(a) * b, F);
}
__device__ __forceinline__ uint32_t addmod(uint32_t a, uint32_t b, const FieldParams& F) {
    uint32_t s = a + b;
    return s >= F.p ? s - F.p : s;
}
__device__ __forceinline__ uint32_t submod(uint32_t a, uint32_t b, const FieldParams& F) {
    return a >= b ? a - b : a + F.p - b;
}
__device__ __forceinline__ uint32_t negmod(uint32_t a, const FieldParams& F) {
    return a ? F.p - a : 0;
}

// a^-1 by Fermat (p prime).  Not on a hot path; a != 0.
__device__ inline uint32_t invmod(uint32_t a, const FieldParams& F) {
    uint32_t e = F.p - 2, r = 1, b = a;
    while (e) {
        if (e & 1) r = mulmod(r, b, F);
        b = mulmod(b, b, F);
        e >>= 1;
    }
    return r;
}

// Montgomery form helpers (odd p): to_mont(x) = x*2^32 mod p.
__device__ __forceinline__ uint32_t to_mont(uint32_t x, const FieldParams& F) {
    return F.odd ? redc(uint64_t(x) * F.r2, F) : x;
}

// y*a - x*b up to the unit 2^-32 (odd p) -- the fraction-free elimination
// step of the GCD kernel.  For p = 2 the unit is 1.
__device__ __forceinline__ uint32_t ff_comb(uint32_t y, uint32_t a, uint32_t negx, uint32_t b,
                                            const FieldParams& F) {
    uint64_t t = mad_wide(negx, b, uint64_t(y) * a);
    if (!F.odd) return uint32_t(t % F.p);
    return redc(t, F);
}

}  // namespace mmm_cu
