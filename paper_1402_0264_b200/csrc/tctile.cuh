// tctile.cuh -- shared pieces of the tensor-core polynomial kernels
// (tcmul.cu products, tcdiv.cu divisions): limb-split block-Toeplitz tiles in
// the UMMA SWIZZLE_128B layout and the TMEM plane accumulator (see tcmul.cu).
#pragma once
#include <cstdint>

#include "common.cuh"
#include "tc.cuh"

namespace mmm_cu {
namespace tct {

constexpr int TCM_T = 256;                 // 8 warps: all build, warp 0 lane 0 issues
constexpr int TCM_MAXN = 4096;             // terms per operand
constexpr int TCM_APAD = 128;              // zero words before a (and after, to 4096 + 256)
constexpr int TCM_AWORDS = TCM_APAD + TCM_MAXN + 256;
constexpr uint32_t TILE = 128 * 128;       // one limb tile of H_d (bytes)
constexpr uint32_t HBUF = 4 * TILE;        // four limb tiles
// B operand: rows 64 v + j (limb v, block j < 32) of a 240-row region whose
// preceding row is zero.  Even d: MMA N = 224 from the region's start; odd d:
// N = 240 from one row earlier (descriptors may start at any 128-byte row: the
// SWIZZLE_128B pattern follows absolute address bits, base_offset 0; measured
// by tools/tc_i8_probe), i.e. every row one later -- the TMEM column offset
// (which must be even) stays d & ~1.
constexpr uint32_t BROWS_E = 224, BROWS_O = 240;
constexpr uint32_t B_PRE = 1024;                         // keeps the region 1024-aligned
constexpr uint32_t B_BYTES = B_PRE + BROWS_O * 128;
// shared layout (bytes, from a 1024-aligned base)
constexpr uint32_t OFF_H = 0;                            // 2 x HBUF
constexpr uint32_t OFF_B = OFF_H + 2 * HBUF;             // B_PRE | 240 rows
constexpr uint32_t OFF_A = OFF_B + B_BYTES;              // u32 a, padded
constexpr uint32_t SMEM_BYTES = OFF_A + TCM_AWORDS * 4 + 1024;



// 4 x 4 byte transpose: out[u] = byte u of w0, w1, w2, w3 (little-endian order)
__device__ __forceinline__ void limb_transpose(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                                               uint32_t& l0, uint32_t& l1, uint32_t& l2,
                                               uint32_t& l3) {
    const uint32_t x0 = __byte_perm(w0, w1, 0x5140), x1 = __byte_perm(w0, w1, 0x7362);
    const uint32_t x2 = __byte_perm(w2, w3, 0x5140), x3 = __byte_perm(w2, w3, 0x7362);
    l0 = __byte_perm(x0, x2, 0x5410);
    l1 = __byte_perm(x0, x2, 0x7632);
    l2 = __byte_perm(x1, x3, 0x5410);
    l3 = __byte_perm(x1, x3, 0x7632);
}

__device__ __forceinline__ void sts128(uint8_t* base, uint32_t off, uint32_t a, uint32_t b,
                                       uint32_t c, uint32_t d) {
    *reinterpret_cast<uint4*>(base + off) = make_uint4(a, b, c, d);
}

// 16 words w[0..15] (element t = 16c + t') of row `row`, chunk c, into the four
// limb tiles at `h` (tile u at h + u * TILE).
__device__ __forceinline__ void put_row_chunk(uint8_t* h, uint32_t tile_stride, uint32_t row,
                                              uint32_t c, const uint32_t (&w)[16]) {
    uint32_t L[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
        limb_transpose(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3], L[0][q], L[1][q],
                       L[2][q], L[3][q]);
    const uint32_t off = tc::sw128(row, 16 * c);
#pragma unroll
    for (int u = 0; u < 4; ++u) sts128(h + u * tile_stride, off, L[u][0], L[u][1], L[u][2], L[u][3]);
}

// Rows 4 rg .. 4 rg + 3, chunk c (elements t in [16c, 16c+16)) of the four limb
// tiles of H_d: row r = 4 rg + k needs a[i0 + k - t'], t' = 0..15,
// i0 = 128 d + 4 rg - 16 c: words a[i0 - 16 .. i0 + 3] (20, 16-byte aligned
// with the pad of 128).
// SWZ: the words are stored with swz_word() (a_pad 128-word aligned): the eight
// lanes of a quarter-warp (one row group, chunks 0..7) read 16-byte slots 64
// bytes apart, a 4-way bank conflict in the plain layout (measured: 12 excess
// wavefronts per load), none with the slots of each 128-byte line XORed by the
// line index.
__device__ __forceinline__ int swz_word(int w) { return w ^ (((w >> 5) & 3) << 2); }
template <bool SWZ = false>
__device__ __forceinline__ void build_unit(uint8_t* hbuf, const uint32_t* a_pad, int d, int rg,
                                           int c) {
    const int i0 = 128 * d + 4 * rg - 16 * c;
    const int w0 = TCM_APAD + i0 - 16;
    const uint4* src = reinterpret_cast<const uint4*>(a_pad + w0);
    uint32_t x[20];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const uint4 v = SWZ ? *reinterpret_cast<const uint4*>(a_pad + swz_word(w0 + 4 * q)) : src[q];
        x[4 * q] = v.x;
        x[4 * q + 1] = v.y;
        x[4 * q + 2] = v.z;
        x[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t wv[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) wv[t] = x[16 + k - t];  // a[i0 + k - t]
        put_row_chunk(hbuf, TILE, uint32_t(4 * rg + k), uint32_t(c), wv);
    }
}

// H_d limb tiles by 256 threads: thread (warp w, lane L) builds rows
// 4 rg .. 4 rg + 3 of chunk c, rg = 4 w + L / 8, c = L % 8 (conflict-free loads
// and swizzled stores).
template <bool SWZ = false>
__device__ __forceinline__ void build_h(uint8_t* hbuf, const uint32_t* a_pad, int d) {
    const int w = threadIdx.x >> 5, L = threadIdx.x & 31;
    build_unit<SWZ>(hbuf, a_pad, d, 4 * w + (L >> 3), L & 7);
}

__device__ __forceinline__ void tmem_st32_zero(uint32_t taddr) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(0u)
        : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}


// w[t] = p[t] for t < 16, words at or past `valid` read as zero; four 16-byte
// loads when p is 16-byte aligned and the 16 words are all valid.
__device__ __forceinline__ void load16(const uint32_t* p, int valid, uint32_t (&w)[16]) {
    if (valid >= 16 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + q);
            w[4 * q] = v.x;
            w[4 * q + 1] = v.y;
            w[4 * q + 2] = v.z;
            w[4 * q + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int t = 0; t < 16; ++t) w[t] = t < valid ? __ldg(p + t) : 0u;
    }
}

// a_pad[base + i] = a[i] for i in [lo, hi) (zero where i >= n), 16-byte loads
// and stores where a and the range allow (lo a multiple of 4).
// SWZ: stored with swz_word() (dst a multiple of 128 words past the swizzle's origin).
template <bool SWZ = false>
__device__ __forceinline__ void stage_words(uint32_t* dst, const uint32_t* a, int lo, int hi, int n,
                                            int tid, int nthreads) {
    if ((reinterpret_cast<uintptr_t>(a) & 15) == 0 && (lo & 3) == 0 &&
        (reinterpret_cast<uintptr_t>(dst + lo) & 15) == 0) {
        for (int i = lo + 4 * tid; i < hi; i += 4 * nthreads) {
            uint4 v;
            if (i + 4 <= n) {
                v = __ldg(reinterpret_cast<const uint4*>(a + i));
            } else {
                v.x = i < n ? __ldg(a + i) : 0u;
                v.y = i + 1 < n ? __ldg(a + i + 1) : 0u;
                v.z = i + 2 < n ? __ldg(a + i + 2) : 0u;
                v.w = i + 3 < n ? __ldg(a + i + 3) : 0u;
            }
            const int is = SWZ ? swz_word(i) : i;
            if (i + 4 <= hi) {
                *reinterpret_cast<uint4*>(dst + is) = v;
            } else {
                const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
                for (int q = 0; i + q < hi; ++q) dst[is + q] = vv[q];
            }
        }
    } else {
        for (int i = lo + tid; i < hi; i += nthreads)
            dst[SWZ ? swz_word(i) : i] = i < n ? __ldg(a + i) : 0u;
    }
}

__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
    return v;
}

// sum_s x_s 2^(8 s) mod p for the seven limb planes (x_s < 2^31)
__device__ __forceinline__ uint32_t combine_planes(const uint32_t (&x)[7], const uint32_t* c_hi,
                                                   const FieldParams& F) {
    uint64_t v = uint64_t(x[0]) + (uint64_t(x[1]) << 8) + (uint64_t(x[2]) << 16) +
                 (uint64_t(x[3]) << 24);
    v += uint64_t(x[4]) * c_hi[0];
    v += uint64_t(x[5]) * c_hi[1];
    v += uint64_t(x[6]) * c_hi[2];
    return reduce(v, F);
}

}  // namespace tct
}  // namespace mmm_cu
