// conv.cuh -- the register-tiled modular convolution engine shared by the
// plain-multiplication, division-update and GCD matrix-apply kernels.
//
// One thread owns R consecutive outputs and walks the terms in blocks of R:
// per block it loads R term words (warp-uniform, LDS.128 broadcast) and R new
// window words (its own, LDS.128), then issues R*R IMAD.WIDE.U32 into 64-bit
// accumulators.  This is the paper's "each thread computes s x s partial
// products from locally staged coefficients" (Alg. 5-7;
// proj/src/multiplication.cpp:85-103 simulates it with s = R), re-expressed
// for registers: the 2R-1 window words slide down by R per block so only R
// are reloaded.  Accumulators are folded (fold(), field.cuh) every
// F.fold_terms products, so a block of R terms costs R*R IMAD.WIDE plus an
// amortised fold.
#pragma once
#include <cstdint>

#include "field.cuh"

namespace mmm_cu {

// acc[r] += sum_{u < nblk*R} sw[u] * sv[base + r - u]
// Requirements: R in {1,2,4,8,16}; for R % 4 == 0: sw 16-byte aligned and
// base % 4 == 3 (so every window reload is one aligned uint4 per 4 words).
// `since` counts products added since the last fold (carried across calls).
template <int R>
__device__ __forceinline__ void conv_accumulate(uint64_t (&acc)[R], const uint32_t* __restrict__ sw,
                                                int nblk, const uint32_t* __restrict__ sv, int base,
                                                uint32_t& since, const FieldParams& F) {
    uint32_t W[2 * R - 1];
#pragma unroll
    for (int j = 0; j < R - 1; ++j) W[R + j] = sv[base + 1 + j];
    for (int blk = 0; blk < nblk; ++blk) {
        const int u0 = blk * R;
        if (since + R > F.fold_terms) {
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = fold(acc[r], F);
            since = 0;
        }
        since += R;
        uint32_t X[R];
        const int lo = base - u0 - (R - 1);
        if constexpr (R % 4 == 0) {
#pragma unroll
            for (int q = 0; q < R / 4; ++q) {
                const uint4 w = *reinterpret_cast<const uint4*>(sv + lo + 4 * q);
                W[4 * q + 0] = w.x;
                W[4 * q + 1] = w.y;
                W[4 * q + 2] = w.z;
                W[4 * q + 3] = w.w;
                const uint4 x = *reinterpret_cast<const uint4*>(sw + u0 + 4 * q);
                X[4 * q + 0] = x.x;
                X[4 * q + 1] = x.y;
                X[4 * q + 2] = x.z;
                X[4 * q + 3] = x.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < R; ++j) {
                W[j] = sv[lo + j];
                X[j] = sw[u0 + j];
            }
        }
#pragma unroll
        for (int t = 0; t < R; ++t)
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = mad_wide(X[t], W[(R - 1) + r - t], acc[r]);
#pragma unroll
        for (int j = R - 2; j >= 0; --j) W[j + R] = W[j];
    }
}

// Fixed trip count NB, no fold: for NB*R <= F.fold_terms the sums cannot
// overflow, so the blocks unroll into straight-line code (all window and term
// loads in flight at once; no per-block fold test or loop branch).  Reads the
// same words as conv_accumulate (sv[base - NB*R + 1 .. base + R - 1]).
template <int R, int NB>
__device__ __forceinline__ void conv_accumulate_fixed(uint64_t (&acc)[R], const uint32_t* __restrict__ sw,
                                                      const uint32_t* __restrict__ sv, int base) {
    static_assert(R % 4 == 0, "conv_accumulate_fixed: R multiple of 4");
    uint32_t W[R * NB + R - 1];  // W[k] = sv[base - NB*R + 1 + k]
    uint32_t X[R * NB];
#pragma unroll
    for (int q = 0; q < NB * R / 4; ++q) {
        const uint4 w = *reinterpret_cast<const uint4*>(sv + base - NB * R + 1 + 4 * q);
        W[4 * q + 0] = w.x;
        W[4 * q + 1] = w.y;
        W[4 * q + 2] = w.z;
        W[4 * q + 3] = w.w;
    }
#pragma unroll
    for (int j = 0; j < R - 1; ++j) W[NB * R + j] = sv[base + 1 + j];
#pragma unroll
    for (int q = 0; q < NB * R / 4; ++q) {
        const uint4 x = *reinterpret_cast<const uint4*>(sw + 4 * q);
        X[4 * q + 0] = x.x;
        X[4 * q + 1] = x.y;
        X[4 * q + 2] = x.z;
        X[4 * q + 3] = x.w;
    }
    // acc[r] += sum_u X[u] * sv[base + r - u], sv[base + r - u] = W[NB*R - 1 + r - u]
#pragma unroll
    for (int u = 0; u < NB * R; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = mad_wide(X[u], W[NB * R - 1 + r - u], acc[r]);
}

// conv_accumulate<4> with straight-line code for the common block counts
// (1, 2, 4, 8) when the terms fit before the next fold.
__device__ __forceinline__ void conv_accumulate4_fast(uint64_t (&acc)[4], const uint32_t* __restrict__ sw,
                                                      int nblk, const uint32_t* __restrict__ sv,
                                                      int base, uint32_t& since,
                                                      const FieldParams& F) {
    if (since + 4u * unsigned(nblk) <= F.fold_terms) {
        since += 4u * unsigned(nblk);
        switch (nblk) {
            case 1: conv_accumulate_fixed<4, 1>(acc, sw, sv, base); return;
            case 2: conv_accumulate_fixed<4, 2>(acc, sw, sv, base); return;
            case 4: conv_accumulate_fixed<4, 4>(acc, sw, sv, base); return;
            case 8: conv_accumulate_fixed<4, 8>(acc, sw, sv, base); return;
            default: since -= 4u * unsigned(nblk); break;
        }
    }
    conv_accumulate<4>(acc, sw, nblk, sv, base, since, F);
}

// conv_accumulate<R> in straight-line groups of 32 terms (R % 4 == 0): one
// fold test per group instead of per block, no loop branch inside a group.
template <int R>
__device__ __forceinline__ void conv_accumulate_grouped(uint64_t (&acc)[R], const uint32_t* __restrict__ sw,
                                                        int nblk, const uint32_t* __restrict__ sv,
                                                        int base, uint32_t& since,
                                                        const FieldParams& F) {
    constexpr int G = 32 / R;  // blocks per group
    if (R % 4 != 0 || G < 1 || F.fold_terms < unsigned(G * R)) {
        conv_accumulate<R>(acc, sw, nblk, sv, base, since, F);
        return;
    }
    int blk = 0;
    for (; blk + G <= nblk; blk += G) {
        if (since + G * R > F.fold_terms) {
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = fold(acc[r], F);
            since = 0;
        }
        conv_accumulate_fixed<R, (G > 0 ? G : 1)>(acc, sw + blk * R, sv, base - blk * R);
        since += G * R;
    }
    if (blk < nblk) conv_accumulate<R>(acc, sw + blk * R, nblk - blk, sv, base - blk * R, since, F);
}

// The fastest variant for the tile: straight-line groups when R % 4 == 0.
template <int R>
__device__ __forceinline__ void conv_accumulate_auto(uint64_t (&acc)[R], const uint32_t* __restrict__ sw,
                                                     int nblk, const uint32_t* __restrict__ sv,
                                                     int base, uint32_t& since, const FieldParams& F) {
    if constexpr (R % 4 == 0)
        conv_accumulate_grouped<R>(acc, sw, nblk, sv, base, since, F);
    else
        conv_accumulate<R>(acc, sw, nblk, sv, base, since, F);
}

}  // namespace mmm_cu
