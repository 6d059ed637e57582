// tcmul.cu -- batched exact polynomial products over Z/pZ on the sm_100a
// integer tensor core (tcgen05.mma kind::i8, u8 x u8 -> s32 in TMEM).
//
// Computes exactly what oracle_mul computes (proj/src/oracle.cpp:8-15),
// f[k] = sum_i a[i] b[k-i] mod p, for every instance of a batch with
// na, nb <= 4096 terms (cfg5's 4096 x 4096 products).
//
// Block Toeplitz form (block size 128).  With
//   H_d[r][t] = a[128 d + r - t]   (0 outside [0, na)),  B_j[t] = b[128 j + t],
// output block c of the product is f[128 c + r] = sum_{d + j = c} (H_d B_j)[r]:
// for each d, one 128 x 128 Toeplitz tile times all of b's blocks -- a GEMM
// with M = 128 (rows r), K = 128 (t), N = b's blocks.  Exactness: residues
// (< 2^31) split into four u8 limbs, a = sum_u 2^(8u) a_u, b = sum_v 2^(8v) b_v;
// the u8 x u8 products accumulate exactly in s32.
//
// Everything accumulates in TMEM.  Plane s = u + v (0..6) holds, for every
// output block c (0..63), column 64 s + c of the 128-lane accumulator:
//   P_s[r][c] = sum_{u+v=s} sum_{d+j=c} (H^u_d B^v_j)[r]   (< 33*4*128*255^2 < 2^31).
// The B operand of d's MMAs lists rows n = 64 v + j (v = 0..3, j < 32: the
// limb blocks of b, zero rows between), so the MMA for limb u of H_d written
// at TMEM column 64 u + d lands (u, v, j) on column 64 (u + v) + (d + j):
// limb-plane and output-block bookkeeping are both done by the tensor core's
// column offset.  MMA D columns must be even: odd d uses a copy of the B
// operand shifted by one row and the column offset d - 1.  At the end,
//   f[128 c + r] = sum_s P_s[r][c] 2^(8 s)  mod p        (one reduction).
//
// Per instance: stage a (smem), build both B copies (limb transpose), zero
// TMEM; then for each d the 4 limb tiles of H_d are built into one of two
// buffers while the tensor core runs the previous d's 16 MMAs (128 x N x 32,
// N = 224 / 240); one thread issues, tcgen05.commit -> mbarrier frees the
// buffer.  Persistent: one CTA per SM walks the batch.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc.cuh"
#include "tctile.cuh"

namespace mmm_cu {

namespace cg = cooperative_groups;

namespace {

using namespace tct;

struct TcArgs {
    const uint32_t* A;
    const uint32_t* B;
    int64_t lda, ldb, ldf;
    int na, nb;
    int64_t count;
    Fan F;
    FieldParams Fp;
    uint32_t c_hi[3];  // 2^32, 2^40, 2^48 mod p
};

// MMM_TC_STATS builds: per-phase clock sums (CTA 0, thread 0) in tcm_stats
__device__ long long tcm_stats[8];

template <bool FAN>
__global__ void __launch_bounds__(TCM_T + 32, 1) tcmul_kernel(TcArgs g) {
    extern __shared__ uint8_t smem_raw[];
    // Aligned through an integer: the tile build then uses generic ST/LD, which
    // measured 6% faster here than LDS/STS while the build's loads were bank
    // conflicted (1.42 vs 1.51 ms for cfg5's products) and the same since the
    // Toeplitz words are stored slot-swizzled (1.157 ms either way: the tile
    // stream runs at the tensor core's rate); tcdiv uses tc::align_smem_1024.
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
    uint8_t* sH = sm + OFF_H;
    uint8_t* sBE = sm + OFF_B + B_PRE;
    uint32_t* a_pad = reinterpret_cast<uint32_t*>(sm + OFF_A);
    __shared__ uint64_t full[2], empty[2];  // tile in buffer b built / its MMAs done
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int na = g.na, nb = g.nb;
    const int mB = (nb + 127) >> 7;
    const int D = (na + 126) / 128 + 1;           // d = 0 .. D-1 (H_d nonzero)
    const int nf = na + nb - 1;
    const int nc = (nf + 127) >> 7;               // output blocks

    // zero the B region and the a pad once (data rows are rewritten per instance)
    for (uint32_t i = tid; i < B_BYTES / 16; i += TCM_T + 32)
        reinterpret_cast<uint4*>(sm + OFF_B)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < TCM_AWORDS; i += TCM_T + 32) a_pad[i] = 0;
    if (warp == 0) tc::tmem_alloc<512>(&tslot);
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&full[b], 1);
            tc::mbar_init(&empty[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = tslot;

    if (warp == TCM_T / 32) {
        // ---- MMA warp: tile after tile, buffer T & 1 (T counts tiles over instances) ----
        constexpr uint32_t ID_E = tc::idesc_u8(128, BROWS_E), ID_O = tc::idesc_u8(128, BROWS_O);
        uint32_t fph[2] = {0, 0};
        uint32_t T = 0;
        for (int64_t inst = blockIdx.x; inst < g.count; inst += gridDim.x)
            for (int d = 0; d < D; ++d, ++T) {
                const int b = T & 1;
                tc::mbar_wait(&full[b], fph[b]);
                fph[b] ^= 1;
                tc::fence_after_sync();
                if (lane == 0) {
                    const uint32_t hb = tc::smem_u32(sH + b * HBUF);
                    const bool odd = d & 1;
                    const uint32_t bb = tc::smem_u32(sBE) - (odd ? 128u : 0u);
                    const uint32_t idesc = odd ? ID_O : ID_E;
                    const uint32_t col = uint32_t(d & ~1);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            tc::mma_u8(tbase + 64 * u + col, tc::desc_sw128(hb + u * TILE + 32 * k),
                                       tc::desc_sw128(bb + 32 * k), idesc, 1u);
                    tc::commit(&empty[b]);
                }
                __syncwarp();
            }
    } else {
        // ---- 8 compute warps: operands in, tiles built, planes out ----
        uint32_t eph[2] = {0, 0};
        int pend[2] = {0, 0};  // handed-off tiles whose MMAs were not yet waited for
        uint32_t T = 0;
        auto free_buf = [&](int b) {
            if (pend[b]) {
                tc::mbar_wait(&empty[b], eph[b]);
                eph[b] ^= 1;
                --pend[b];
            }
        };
        auto bar = [] { asm volatile("bar.sync 1, 256;" ::: "memory"); };
        long long t_pro = 0, t_loop = 0, t_epi = 0, t_mmawait = 0, t0, t1;
        // Rows whose words can be moved as whole 16-byte groups: each thread then holds
        // the next instance's share of a and b (4 + 4 groups) in registers, loaded while
        // the current instance's tiles run, so the prologue does not wait for HBM.
        const bool pre_ok = (reinterpret_cast<uintptr_t>(g.A) & 15) == 0 &&
                            (reinterpret_cast<uintptr_t>(g.B) & 15) == 0 && (g.lda & 3) == 0 &&
                            (g.ldb & 3) == 0 && (na & 3) == 0 && (nb & 3) == 0;
        uint4 pa[4], pb[4];
        auto prefetch_rows = [&](int64_t which) {
            const uint32_t* a = g.A + which * g.lda;
            const uint32_t* b = g.B + which * g.ldb;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int ia = 4 * tid + 4 * TCM_T * q, ib = 16 * tid + 4 * q;
                pa[q] = ia < na ? __ldg(reinterpret_cast<const uint4*>(a + ia)) : make_uint4(0, 0, 0, 0);
                pb[q] = ib < nb ? __ldg(reinterpret_cast<const uint4*>(b + ib)) : make_uint4(0, 0, 0, 0);
            }
        };
        if (pre_ok && int64_t(blockIdx.x) < g.count) prefetch_rows(blockIdx.x);
        for (int64_t inst = blockIdx.x; inst < g.count; inst += gridDim.x) {
            t0 = clock64();
            const uint32_t* a = g.A + inst * g.lda;
            const uint32_t* b = g.B + inst * g.ldb;
            if (pre_ok) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int ia = 4 * tid + 4 * TCM_T * q;
                    if (ia < na) *reinterpret_cast<uint4*>(a_pad + TCM_APAD + swz_word(ia)) = pa[q];
                }
            } else {
                stage_words<true>(a_pad + TCM_APAD, a, 0, na, na, tid, TCM_T);
            }
            // B rows 64 v + j; unit = (j, chunk c)
            for (int u = tid; u < mB * 8; u += TCM_T) {
                const int j = u >> 3, c = u & 7;
                uint32_t wv[16];
                if (pre_ok) {  // u == tid: words b[16 u .. 16 u + 15]
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        wv[4 * q] = pb[q].x;
                        wv[4 * q + 1] = pb[q].y;
                        wv[4 * q + 2] = pb[q].z;
                        wv[4 * q + 3] = pb[q].w;
                    }
                } else {
                    load16(b + 128 * j + 16 * c, nb - (128 * j + 16 * c), wv);
                }
                uint32_t L[4][4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    limb_transpose(wv[4 * q], wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3], L[0][q],
                                   L[1][q], L[2][q], L[3][q]);
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    sts128(sBE, tc::sw128(64 * v + j, 16 * c), L[v][0], L[v][1], L[v][2], L[v][3]);
            }
            if (pre_ok && inst + gridDim.x < g.count) prefetch_rows(inst + gridDim.x);
            if (warp < 4) {
#pragma unroll
                for (int c0 = 0; c0 < 512; c0 += 32)
                    tmem_st32_zero(tbase + (uint32_t(warp * 32) << 16) + c0);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            bar();  // a staged
            t1 = clock64();
            t_pro += t1 - t0;
            t0 = t1;
            for (int d = 0; d < D; ++d, ++T) {
                const int bb = T & 1;
                const long long tw = clock64();
                free_buf(bb);
                t_mmawait += clock64() - tw;
                build_h<true>(sH + bb * HBUF, a_pad, d);
                tc::fence_async_smem();
                tc::fence_before_sync();
                bar();
                if (tid == 0) tc::mbar_arrive(&full[bb]);
                ++pend[bb];
            }
            free_buf(0);  // every MMA of this instance is done
            free_buf(1);
            tc::fence_after_sync();
            t1 = clock64();
            t_loop += t1 - t0;
            t0 = t1;
            // ---- epilogue: warps w and w+4 share lanes 32 (w % 4) .. +31 ----
            {
                const int r = 32 * (warp & 3) + lane;
                const int cbeg = (warp >> 2) * 32;
                const uint32_t lane_addr = tbase + (uint32_t(32 * (warp & 3)) << 16);
                const FieldParams& Fp = g.Fp;
                const int64_t fb = inst * g.ldf;
                for (int c0 = cbeg; c0 < cbeg + 32 && c0 < nc; c0 += 8) {
                    uint32_t x[7][8];
#pragma unroll
                    for (int s = 0; s < 7; ++s) tmem_ld8(lane_addr + 64 * s + c0, x[s]);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int k = 128 * (c0 + e) + r;
                        uint64_t v = uint64_t(x[0][e]) + (uint64_t(x[1][e]) << 8) +
                                     (uint64_t(x[2][e]) << 16) + (uint64_t(x[3][e]) << 24);
                        v += uint64_t(x[4][e]) * g.c_hi[0];
                        v += uint64_t(x[5][e]) * g.c_hi[1];
                        v += uint64_t(x[6][e]) * g.c_hi[2];
                        if (k < nf) fan_store<FAN>(g.F, fb + k, reduce(v, Fp));
                    }
                }
            }
            tc::fence_before_sync();
            bar();  // TMEM read before the next instance zeroes it
            tc::fence_after_sync();
            t_epi += clock64() - t0;
        }
        if (blockIdx.x == 0 && tid == 0) {
            tcm_stats[0] = t_pro;
            tcm_stats[1] = t_loop;
            tcm_stats[2] = t_epi;
            tcm_stats[3] = t_mmawait;
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) tc::tmem_free<512>(tbase);
}

// ---- one large product split over the SMs (cfg1: 2^14 x 2^14) -------------
// a and b cut into segments of <= 4096 terms; work item = (segment of a,
// segment of b, a range of <= 32 consecutive tiles d of that segment pair).
// An item accumulates its tiles in the TMEM planes exactly like a batch
// instance (column offset d - d0), then adds its reduced outputs into a u64
// accumulator (RED.ADD.U64; up to a few dozen residues per word); after a grid
// barrier every thread finalises a slice: f = acc mod p, acc = 0 (ZeroBuf).
struct TcSplitArgs {
    const uint32_t* a;
    const uint32_t* b;
    int na, nb, nf;
    int segA, segB, dpr;          // segments of a / b, tiles per item
    int rA;                        // items per segment pair (max over a's segments)
    int items;
    unsigned long long* acc;
    Fan F;
    FieldParams Fp;
    uint32_t c_hi[3];
};

struct Item {
    int ia, ib, d0, d1, na_i, nb_j;
};

__device__ __forceinline__ bool decode_item(const TcSplitArgs& g, int w, Item& it) {
    const int pr = w / g.rA, r = w % g.rA;
    it.ia = pr / g.segB;
    it.ib = pr % g.segB;
    it.na_i = min(TCM_MAXN, g.na - TCM_MAXN * it.ia);
    it.nb_j = min(TCM_MAXN, g.nb - TCM_MAXN * it.ib);
    const int D = (it.na_i + 126) / 128 + 1;
    it.d0 = r * g.dpr;
    it.d1 = min(D, it.d0 + g.dpr);
    return it.d0 < it.d1;
}

__global__ void __launch_bounds__(TCM_T + 32, 1) tcmul_split_kernel(TcSplitArgs g) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = tc::align_smem_1024(smem_raw);
    uint8_t* sH = sm + OFF_H;
    uint8_t* sBE = sm + OFF_B + B_PRE;
    uint32_t* a_pad = reinterpret_cast<uint32_t*>(sm + OFF_A);
    __shared__ uint64_t full[2], empty[2];
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    for (uint32_t i = tid; i < B_BYTES / 16; i += TCM_T + 32)
        reinterpret_cast<uint4*>(sm + OFF_B)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < TCM_AWORDS; i += TCM_T + 32) a_pad[i] = 0;
    if (warp == 0) tc::tmem_alloc<512>(&tslot);
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&full[b], 1);
            tc::mbar_init(&empty[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = tslot;

    if (warp == TCM_T / 32) {  // MMA warp
        constexpr uint32_t ID_E = tc::idesc_u8(128, BROWS_E), ID_O = tc::idesc_u8(128, BROWS_O);
        uint32_t fph[2] = {0, 0};
        uint32_t T = 0;
        for (int w = blockIdx.x; w < g.items; w += gridDim.x) {
            Item it;
            if (!decode_item(g, w, it)) continue;
            for (int d = it.d0; d < it.d1; ++d, ++T) {
                const int b = T & 1;
                tc::mbar_wait(&full[b], fph[b]);
                fph[b] ^= 1;
                tc::fence_after_sync();
                if (lane == 0) {
                    const int e = d - it.d0;
                    const uint32_t hb = tc::smem_u32(sH + b * HBUF);
                    const bool odd = e & 1;
                    const uint32_t bb = tc::smem_u32(sBE) - (odd ? 128u : 0u);
                    const uint32_t idesc = odd ? ID_O : ID_E;
                    const uint32_t col = uint32_t(e & ~1);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            tc::mma_u8(tbase + 64 * u + col, tc::desc_sw128(hb + u * TILE + 32 * k),
                                       tc::desc_sw128(bb + 32 * k), idesc, 1u);
                    tc::commit(&empty[b]);
                }
                __syncwarp();
            }
        }
    } else {
        uint32_t eph[2] = {0, 0};
        int pend[2] = {0, 0};
        uint32_t T = 0;
        auto free_buf = [&](int b) {
            if (pend[b]) {
                tc::mbar_wait(&empty[b], eph[b]);
                eph[b] ^= 1;
                --pend[b];
            }
        };
        auto bar = [] { asm volatile("bar.sync 1, 256;" ::: "memory"); };
        const uint32_t lane_addr = tbase + (uint32_t(32 * (warp & 3)) << 16);
        long long t0 = clock64(), sp[4] = {0, 0, 0, 0};
        for (int w = blockIdx.x; w < g.items; w += gridDim.x) {
            Item it;
            if (!decode_item(g, w, it)) continue;
            const long long ti = clock64();
            const uint32_t* a = g.a + int64_t(TCM_MAXN) * it.ia;
            const uint32_t* b = g.b + int64_t(TCM_MAXN) * it.ib;
            // the window of a the tiles d0..d1-1 read: [128 d0 - 128, 128 d1)
            const int lo = max(0, 128 * it.d0 - 128), hi = min(TCM_MAXN + 128, 128 * it.d1);
            stage_words<true>(a_pad + TCM_APAD, a, lo, hi, it.na_i, tid, TCM_T);
            const int mB = (it.nb_j + 127) >> 7;
            for (int u = tid; u < 32 * 8; u += TCM_T) {  // all 32 block rows (zeros past mB)
                const int j = u >> 3, c = u & 7;
                uint32_t wv[16];
                load16(b + 128 * j + 16 * c, j < mB ? it.nb_j - (128 * j + 16 * c) : 0, wv);
                uint32_t L[4][4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    limb_transpose(wv[4 * q], wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3], L[0][q],
                                   L[1][q], L[2][q], L[3][q]);
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    sts128(sBE, tc::sw128(64 * v + j, 16 * c), L[v][0], L[v][1], L[v][2], L[v][3]);
            }
            if (warp < 4) {
#pragma unroll
                for (int c0 = 0; c0 < 512; c0 += 32) tmem_st32_zero(lane_addr + c0);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            bar();
            const long long tl = clock64();
            sp[0] += tl - ti;
            for (int d = it.d0; d < it.d1; ++d, ++T) {
                const int bb = T & 1;
                free_buf(bb);
                build_h<true>(sH + bb * HBUF, a_pad, d);
                tc::fence_async_smem();
                tc::fence_before_sync();
                bar();
                if (tid == 0) tc::mbar_arrive(&full[bb]);
                ++pend[bb];
            }
            free_buf(0);
            free_buf(1);
            tc::fence_after_sync();
            const long long te = clock64();
            sp[1] += te - tl;
            // outputs of this item: blocks d0 + e, e < (d1 - d0) + mB, of segment pair (ia, ib)
            {
                const int r = 32 * (warp & 3) + lane;
                const int ne = (it.d1 - it.d0) + mB;
                const int64_t kb = int64_t(TCM_MAXN) * (it.ia + it.ib) + 128 * it.d0 + r;
                for (int e0 = (warp >> 2) * 8; e0 < ne; e0 += 16) {
                    uint32_t x[7][8];
#pragma unroll
                    for (int s = 0; s < 7; ++s) tmem_ld8(lane_addr + 64 * s + e0, x[s]);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int64_t k = kb + 128 * (e0 + e);
                        if (e0 + e < ne && k < g.nf) {
                            const uint32_t xs[7] = {x[0][e], x[1][e], x[2][e], x[3][e], x[4][e],
                                                    x[5][e], x[6][e]};
                            atomicAdd(g.acc + k,
                                      (unsigned long long)combine_planes(xs, g.c_hi, g.Fp));
                        }
                    }
                }
            }
            tc::fence_before_sync();
            bar();  // TMEM read before the next item zeroes it
            tc::fence_after_sync();
            sp[2] += clock64() - te;
        }
        if (blockIdx.x == 0 && tid == 0) {
            tcm_stats[4] = sp[0];
            tcm_stats[5] = sp[1];
            tcm_stats[6] = sp[2];
            tcm_stats[7] = clock64() - t0;
        }
    }
    // every item's additions are in acc: finalise (f = acc mod p, acc back to zero)
    __threadfence();
    cg::this_grid().sync();
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + tid; k < g.nf; k += stride) {
        const unsigned long long v = __ldcg(g.acc + k);
        g.acc[k] = 0ull;
        fan_store<true>(g.F, k, reduce(v, g.Fp));
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) tc::tmem_free<512>(tbase);
}

}  // namespace

// Routing (mul.cu, divmod.cu): an explicit program parameter s >= 1 selects the
// paper's s-parameterised CUDA-core kernel; s <= 0 ("auto") lets the library
// take the tensor core where it pays.  MMM_MUL_TC / MMM_DIV_TC = 1 force the
// tensor core wherever the shape allows (tests), 0 forbids it.
bool tc_route(const char* env, int64_t s, bool shape_ok, bool worth) {
    if (const char* e = getenv(env)) return atoi(e) != 0 && shape_ok;
    return s <= 0 && shape_ok && worth;
}

bool tcmul_supported(int64_t na, int64_t nb, int64_t count, int64_t s) {
    const bool shape = na >= 1 && nb >= 1 && na <= TCM_MAXN && nb <= TCM_MAXN;
    return tc_route("MMM_MUL_TC", s, shape,
                    na >= 512 && nb >= 512 && double(na) * double(nb) * double(count) >= 1.0e9);
}

void launch_tcmul_batched(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                          const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, Fan Fo,
                          int64_t ldf, cudaStream_t st) {
    if (count <= 0) return;
    if (na < 1 || nb < 1 || na > TCM_MAXN || nb > TCM_MAXN)
        throw Error(ST_INVALID, "tensor-core product: operands of 1..4096 terms");
    TcArgs g{};
    g.A = A;
    g.B = B;
    g.lda = lda;
    g.ldb = ldb;
    g.ldf = ldf;
    g.na = int(na);
    g.nb = int(nb);
    g.count = count;
    g.F = Fo;
    g.Fp = F;
    for (int s = 0; s < 3; ++s) {
        uint64_t x = 1;
        for (int e = 0; e < 32 + 8 * s; ++e) x = (x * 2) % F.p;
        g.c_hi[s] = uint32_t(x);
    }
    auto kern = Fo.n > 1 ? tcmul_kernel<true> : tcmul_kernel<false>;
    MMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES)));
    const int blocks = int(std::min<int64_t>(count, sm_count()));
    kern<<<blocks, TCM_T + 32, SMEM_BYTES, st>>>(g);
    check_launch("tcmul_kernel", dim3(blocks), dim3(TCM_T + 32));
    if (getenv("MMM_TC_STATS")) {
        long long h[8];
        MMM_CUDA(cudaMemcpyFromSymbolAsync(h, tcm_stats, sizeof(h), 0, cudaMemcpyDeviceToHost, st));
        MMM_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "tcmul stats (CTA 0): prologue=%lld loop=%lld epilogue=%lld mma_wait=%lld cycles\n",
                h[0], h[1], h[2], h[3]);
    }
}

bool tcmul_single_supported(int64_t na, int64_t nb, int64_t s) {
    return tc_route("MMM_MUL_TC", s, na >= 1 && nb >= 1,
                    double(na) * double(nb) >= 3.0e7 && na >= 512 && nb >= 512);
}

// One product f = a * b (all na + nb - 1 words) on the tensor core, split over
// the SMs (tcmul_split_kernel).
void launch_tcmul_single(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b,
                         int64_t nb, Fan Fo, cudaStream_t st) {
    if (na < 1 || nb < 1) throw Error(ST_INVALID, "tensor-core product: empty operand");
    if (na + nb > (int64_t(1) << 30)) throw Error(ST_INVALID, "tensor-core product: too long");
    TcSplitArgs g{};
    g.a = a;
    g.b = b;
    g.na = int(na);
    g.nb = int(nb);
    g.nf = int(na + nb - 1);
    g.segA = int(ceil_div(na, TCM_MAXN));
    g.segB = int(ceil_div(nb, TCM_MAXN));
    const int Dmax = (int(std::min<int64_t>(na, TCM_MAXN)) + 126) / 128 + 1;
    const int64_t tiles = int64_t(g.segA) * g.segB * Dmax;
    const int sms = sm_count();
    g.dpr = int(std::max<int64_t>(1, std::min<int64_t>(32, ceil_div(tiles, sms))));
    g.rA = (Dmax + g.dpr - 1) / g.dpr;
    g.items = g.segA * g.segB * g.rA;
    g.F = Fo;
    g.Fp = F;
    for (int s = 0; s < 3; ++s) {
        uint64_t x = 1;
        for (int e = 0; e < 32 + 8 * s; ++e) x = (x * 2) % F.p;
        g.c_hi[s] = uint32_t(x);
    }
    g.acc = zero_buf_acquire(size_t(g.nf), st);
    MMM_CUDA(cudaFuncSetAttribute(tcmul_split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(SMEM_BYTES)));
    const int blocks = std::min(g.items, sms);
    void* params[] = {&g};
    MMM_CUDA(cudaLaunchCooperativeKernel((void*)tcmul_split_kernel, dim3(blocks), dim3(TCM_T + 32),
                                         params, SMEM_BYTES, st));
    check_launch("tcmul_split_kernel", dim3(blocks), dim3(TCM_T + 32));
    zero_buf_release(st);
    if (getenv("MMM_TC_STATS")) {
        long long h[8];
        MMM_CUDA(cudaMemcpyFromSymbolAsync(h, tcm_stats, sizeof(h), 0, cudaMemcpyDeviceToHost, st));
        MMM_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "tcmul_split stats (CTA 0): items=%d per_item_tiles=%d stage+B=%lld tiles=%lld "
                "epilogue=%lld total_to_sync=%lld cycles\n", g.items, g.dpr, h[4], h[5], h[6], h[7]);
    }
}

}  // namespace mmm_cu
