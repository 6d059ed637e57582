// tcdiv.cu -- batched long division over Z/pZ on the sm_100a integer tensor
// core: the paper's blocked division (proj/src/division.cpp:81-176, s heads
// retired per step) with s = 128 and the remainder update on tcgen05.
//
// Computes exactly oracle_divmod (proj/src/oracle.cpp:51-67): with
// A' = rev(a), B' = rev(b), mu = na - nb + 1, the reversed quotient is the
// power-series quotient Q = A' / B' mod X^mu, and the remainder is
// r[i] = a[i] - (Q B')[na - 1 - i] for i < nb - 1.  Eliminating 128 heads at
// a time (block K of Q):
//   E_K = block K of (A' - sum_{I<K} Q_I X^(128 I) B'),
//   Q_K = E_K * h mod X^128,   h = B'^-1 mod X^128   (computed once),
// bit-identical to the oracle's head-by-head loop (its zero-head skip is the
// same arithmetic: a zero head gives a zero quotient word).
//
// The running product sum_I Q_I X^(128 I) B' is the block-Toeplitz GEMM of
// tcmul.cu with Q on the Toeplitz side: tile H_K (Q_K below the diagonal,
// Q_{K-1} above) times all of B' goes into the seven TMEM limb planes.  The
// tensor core runs two tiles behind the chain, so when block K is read back
// (S_K) the planes hold tiles <= K-2 and the rest of block K is on the CUDA
// cores:  E_K = A'_K - S_K - T_B1 Q_{K-1} - L_K,  with
//   T_B1[r][m] = B'[128 + r - m]   (Q_{K-1}'s terms in block K: tile K-1's
//                                   lower part against B'_1, tile K's upper
//                                   part against B'_0),
//   L_K[r] = sum_{m > r} Q_{K-2}[m] B'[256 + r - m]   (tile K-1's upper part
//                                   against B'_1: Q_{K-2}'s late terms).
// With Z_K = A'_K - S_K - L_K that is one product per step on the chain:
//   Q_K = T_h Z_K - M Q_{K-1},   M = T_h T_B1   (T_h: lower-triangular
//   Toeplitz of h), where -M (128 x 128, per instance) sits in the compute
// threads' registers -- M[r][m] = M[r-1][m-1] + h[r] B'[128 - m] builds it in
// one diagonal walk per instance -- and -M Q_{K-1} (phase A) runs as soon as
// Q_{K-1} is out, T_h Z_K (phase B) once S_K has been read.  T_h is lower
// triangular and L's matrix U (L_{K+1} = U Q_{K-1}) strictly upper, so the
// two share one 128 x 128 pass: a thread whose 4 x 16 block lies above the
// diagonal runs phase B's instruction stream on (B', Q_{K-1}) instead of
// (h, Z_K); only the diagonal blocks' upper halves (<= 15 terms per row) are
// formed separately (8 MACs per thread in phase A).  After
// the last block one more tile completes Q B' and the remainder comes out of
// TMEM in one pass.  Warps: 8 compute (the chain, the planes' reads, the
// remainder), 3 builders (tiles; the next instance's h by Newton) and one
// issuer (warp 11, one lane: each tile's 16 UMMAs once the tile is written and
// the compute warps have read the block it would disturb -- the issues block
// ~1.8k cycles per tile on the tensor core's queue, which stalled the builders
// while a builder lane issued).  Shapes: na <= 8192, nb <= 4096 (cfg5).
// (Measured alternatives, tools/ab.py on cfg5: L on the builder
// warps 3.44 ms; a 13th warp puts four warps on one SMSP, i.e. <= 128
// registers, too few for M in registers; polling hand-offs, a tile build split
// at the diagonal, byte-window tile rows: all slower than the 2.46 ms here.)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc.cuh"
#include "tctile.cuh"

namespace mmm_cu {

namespace {

using namespace tct;

constexpr int TCD_T = 256;    // compute warps 0-7: the chain
constexpr int TCD_BLD = 96;   // builder warps 8-10: the tiles
constexpr int TCD_ALL = TCD_T + TCD_BLD + 32;  // + warp 11: one lane issues the tiles' UMMAs
                                                // (twelve warps: three per SMSP, up to 168 registers)
constexpr int TCD_MAXA = 8192;
constexpr int TCD_QPAD = 256;                           // zero words before Q
constexpr int TCD_QWORDS = TCD_QPAD + TCD_MAXA + 256;   // Q, padded
// shared layout (bytes, 1024-aligned base)
constexpr uint32_t D_OFF_H = 0;                           // two H buffers (4 limb tiles each)
constexpr uint32_t D_OFF_B = D_OFF_H + 2 * HBUF;          // B_PRE | 240 rows (tctile.cuh)
constexpr uint32_t D_OFF_Q = D_OFF_B + B_BYTES;           // u32 Q (padded)
constexpr uint32_t D_OFF_SM = D_OFF_Q + TCD_QWORDS * 4;   // small arrays
constexpr uint32_t D_SMALL = 256 + 2 * 256 + 128 + 128 + 1024 + 128 + 256 + 1024 + 128 + 256 + 128 + 1024;
// B'[0..256), h ping-pong (each: 128 zeros, h), Z, B' (Montgomery), parts, tmp | builders:
// B'[0..256), parts, tmp | B'[128..256) + 128 zeros, L_{K+1}, L_{K+2}'s partials [8][128]
constexpr uint32_t D_SMEM_BYTES = D_OFF_SM + D_SMALL * 4 + 1024;

struct TcDivArgs {
    const uint32_t* A;
    const uint32_t* B;
    int64_t lda, ldb, ldq, ldr;
    int na, nb;
    int64_t count;
    Fan Q, R;
    FieldParams Fp;
    uint32_t c_hi[3];
};

// lazily reduced dot-product accumulator
struct Acc {
    uint64_t v = 0;
    uint32_t since = 0;
    __device__ __forceinline__ void add(uint32_t x, uint32_t y, const FieldParams& F) {
        if (++since > F.fold_terms) {
            v = fold(v, F);
            since = 1;
        }
        v = mad_wide(x, y, v);
    }
};

// Partial sums of y[i] = sum_{t<T} X[i - t] W[t] (i < n; n % 4 == 0, T % 16 == 0,
// X 16-byte aligned and defined -- zero where the product has no term -- on
// [-T, n)).  Thread (row group g: rows 4g..4g+3, t-part p: t in [16p, 16p+16))
// keeps the four rows' X windows in registers and slides them 4 terms per
// 16-byte load; W[t] is a broadcast.  part[p * n + i] = partial, reduced.
// FAST: odd p with fold_terms >= 16 (no folds inside the 16-term blocks, no p = 2 branch).
template <bool FAST = false>
__device__ __forceinline__ void toeplitz_partials(const uint32_t* X, const uint32_t* W, int n,
                                                  int T, uint32_t* part, const FieldParams& F,
                                                  int tid = -1) {
    const int ng = n >> 2, np = T >> 4;
    if (tid < 0) tid = threadIdx.x;
    if (tid >= ng * np) return;
    const int g = tid % ng, p = tid / ng, r0 = 4 * g, t0 = 16 * p;
    uint4 cv = *reinterpret_cast<const uint4*>(X + r0 - t0);
    uint32_t cur[4] = {cv.x, cv.y, cv.z, cv.w};  // X[r0 - t + k]
    uint64_t acc[4] = {0, 0, 0, 0};
    const uint32_t ft = F.fold_terms;
#pragma unroll
    for (int jb = 0; jb < 4; ++jb) {
        const int t = t0 + 4 * jb;
        const uint4 nv = *reinterpret_cast<const uint4*>(X + r0 - t - 4);
        const uint4 wv = *reinterpret_cast<const uint4*>(W + t);
        const uint32_t z[8] = {nv.x, nv.y, nv.z, nv.w, cur[0], cur[1], cur[2], cur[3]};
        const uint32_t w4[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                acc[k] = mad_wide(z[4 + k - jj], w4[jj], acc[k]);
                if (!FAST && ft < 4) acc[k] = fold(acc[k], F);
            }
        }
        if (!FAST && ft >= 4 && ft < 16)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] = fold(acc[k], F);
        cur[0] = nv.x;
        cur[1] = nv.y;
        cur[2] = nv.z;
        cur[3] = nv.w;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) part[p * n + r0 + k] = reduce_t<FAST>(acc[k], F);
}

// y[i] = sum over the T/16 partials, mod p (threads i < n).
template <bool FAST = false>
__device__ __forceinline__ uint32_t partials_sum(const uint32_t* part, int n, int T, int i,
                                                 const FieldParams& F) {
    uint64_t v = 0;
    for (int p = 0; p < (T >> 4); ++p) v += part[p * n + i];
    return reduce_t<FAST>(v, F);
}

// h = B'^-1 mod X^128 by Newton doubling (h_{2k} = h_k - X^k (h_k e mod X^k),
// e = coefficients [k, 2k) of B' h_k), by the `nt` threads of a group (local id
// ltid) synchronised by `sync`.  bp: B'[0..256); hs: 128 zeros before h.
// One doubling h_k -> h_{2k} (k = 1, 2, ..., 64; h[0] set before k = 1) by the
// `nt` threads of a group (local id ltid) synchronised by `sync`:
// h_{2k} = h_k - X^k (h_k e mod X^k), e = coefficients [k, 2k) of B' h_k.
// bp: B'[0..256); hs: 128 zeros before h.
template <class Sync>
__device__ __forceinline__ void newton_step(const uint32_t* bp, uint32_t* hs, uint32_t* part,
                                            uint32_t* tmp, int ltid, const FieldParams& F, int k,
                                            Sync sync) {
    if (k < 16) {
        if (ltid < k) {
            Acc e;
            for (int m = 0; m < k; ++m) e.add(bp[k + ltid - m], hs[m], F);
            tmp[ltid] = reduce(e.v, F);
        }
        sync();
        if (ltid < k) {
            Acc q;
            for (int m = 0; m <= ltid; ++m) q.add(hs[ltid - m], tmp[m], F);
            hs[k + ltid] = negmod(reduce(q.v, F), F);
        }
        sync();
        return;
    }
    toeplitz_partials(bp + k, hs, k, k, part, F, ltid);  // sliding products
    sync();
    if (ltid < k) tmp[ltid] = partials_sum(part, k, k, ltid, F);
    sync();
    toeplitz_partials(hs, tmp, k, k, part, F, ltid);  // h[i-m], zero for i < m
    sync();
    if (ltid < k) hs[k + ltid] = negmod(partials_sum(part, k, k, ltid, F), F);
    sync();
}

__device__ long long tcd_stats[16];
// Phase clocks (CTA 0) for tuning: build with -DTCD_STATS=1 and run with MMM_TC_STATS=1.
#ifndef TCD_STATS
#define TCD_STATS 0
#endif
__device__ __forceinline__ long long tcd_clock() { return TCD_STATS ? clock64() : 0; }
#define TCD_T0() const long long _t0 = tcd_clock()
#define TCD_ACC(i) \
    if (TCD_STATS) st[i] += clock64() - _t0

template <bool FAN, bool FAST>
__global__ void __maxnreg__(168) tcdiv_kernel(TcDivArgs g) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = tc::align_smem_1024(smem_raw);
    uint8_t* sH = sm + D_OFF_H;
    uint8_t* sBE = sm + D_OFF_B + B_PRE;
    uint32_t* q_pad = reinterpret_cast<uint32_t*>(sm + D_OFF_Q);
    uint32_t* qz = q_pad + TCD_QPAD;                               // Q[0] (Q[-256..-1] = 0)
    uint32_t* bp01 = reinterpret_cast<uint32_t*>(sm + D_OFF_SM);  // B'[0..256)
    uint32_t* hsp = bp01 + 256;                                   // [2][256]: 128 zeros, then h
    uint32_t* sS = hsp + 512;                                     // planes' block K+1
    uint32_t* sE = sS + 128;
    uint32_t* part = sE + 128;                                    // [8][128] partial sums
    uint32_t* tmp = part + 1024;
    uint32_t* bpB = tmp + 128;                                    // builders: next B'[0..256)
    uint32_t* partB = bpB + 256;
    uint32_t* tmpB = partB + 1024;
    uint32_t* bnc = tmpB + 128;  // B'[128..256), then 128 zeros
    uint32_t* lateb = bnc + 256;  // L_{K+1} (see step K)
    uint32_t* partL = lateb + 128;  // [8][128] partials of L_{K+2}
    __shared__ uint64_t full[2], empty[2], qready[2], built[2], hready;
    __shared__ long long issue_ts[2], full_ts[2];
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const FieldParams F = g.Fp;
    const int na = g.na, nb = g.nb;
    const int mu = na - nb + 1;
    const int mB = (nb + 127) >> 7;
    const int Kq = (mu + 127) >> 7;  // quotient blocks; tiles d = 0 .. Kq

    for (uint32_t i = tid; i < B_BYTES / 16; i += TCD_ALL)
        reinterpret_cast<uint4*>(sm + D_OFF_B)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < TCD_QWORDS; i += TCD_ALL) q_pad[i] = 0;
    for (int i = tid; i < 128; i += TCD_ALL) {
        hsp[i] = 0;
        hsp[256 + i] = 0;
    }
    if (warp == 0) tc::tmem_alloc<512>(&tslot);
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&full[b], 4);  // compute warps 0-3, once their rows are read
            tc::mbar_init(&built[b], 1);
            tc::mbar_init(&empty[b], 1);
            tc::mbar_init(&qready[b], 1);
        }
        tc::mbar_init(&hready, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = tslot;

    if (warp >= TCD_T / 32 && warp < (TCD_T + TCD_BLD) / 32) {
        // ---- builder warps: tile K (Q_K lower, Q_{K-1} upper) into buffer T & 1,
        //      while the compute warps run the next step's correction product ----
        // They also compute h = B'^-1 mod X^128 of the instance after the
        // current one while the compute warps finish it (the first instance:
        // up front), into the other half of the h ping-pong.
        const int bt = tid - TCD_T;
        uint32_t qph[2] = {0, 0}, eph[2] = {0, 0};
        long long bst[4] = {0, 0, 0, 0};
        uint32_t T = 0;
        auto bsync = [] { asm volatile("bar.sync 2, %0;" ::"n"(TCD_BLD) : "memory"); };
        // B'[0..256) of instance `which` into bpB and h[0] of its inverse
        auto inverse_begin = [&](int64_t which, uint32_t* hsn) {
            const uint32_t* bb = g.B + which * g.ldb;
            for (int t = bt; t < 256; t += TCD_BLD) bpB[t] = t < nb ? __ldg(bb + (nb - 1 - t)) : 0u;
            bsync();
            if (bt == 0) hsn[0] = invmod(bpB[0], F);
            bsync();
        };
        int ip = 0;
        for (int64_t inst = blockIdx.x; inst < g.count; inst += gridDim.x, ++ip) {
            uint32_t* hsn = hsp + 256 * ((ip + 1) & 1) + 128;  // the next instance's h
            const bool next = inst + gridDim.x < g.count;
            if (ip == 0) {  // the first instance's inverse, up front
                uint32_t* hs0 = hsp + 128;
                inverse_begin(inst, hs0);
                for (int k = 1; k < 128; k <<= 1) newton_step(bpB, hs0, partB, tmpB, bt, F, k, bsync);
                if (bt == 0) tc::mbar_arrive(&hready);
            }
            if (next) inverse_begin(inst + gridDim.x, hsn);
            int kn = 1;  // the next instance's Newton: one doubling after each tile
            for (int K = 0; K <= Kq; ++K, ++T) {
                const int b = T & 1;
                long long tb = tcd_clock();
                tc::mbar_wait(&qready[b], qph[b]);  // Q_K (and Q_{K-1}) published
                qph[b] ^= 1;
                if (T >= 2) {  // the buffer's previous tile (T - 2) is done
                    tc::mbar_wait(&empty[b], eph[b]);
                    eph[b] ^= 1;
                }
                bst[0] += tcd_clock() - tb;
                tb = tcd_clock();
                const int wb = bt >> 5, L = bt & 31;
                // eight warp-units of 4 row groups x 8 chunks over the builder warps
                for (int wu = wb; wu < 8; wu += TCD_BLD / 32)
                    build_unit<true>(sH + b * HBUF, qz - TCM_APAD, K, 4 * wu + (L >> 3), L & 7);
                tc::fence_async_smem();
                bsync();
                bst[1] += tcd_clock() - tb;
                tb = tcd_clock();
                if (bt == 0) tc::mbar_arrive(&built[b]);  // warp 11 issues tile K
                bst[2] += tcd_clock() - tb;
                tb = tcd_clock();
                if (next && kn < 128) {
                    newton_step(bpB, hsn, partB, tmpB, bt, F, kn, bsync);
                    kn <<= 1;
                    if (kn == 128 && bt == 0) tc::mbar_arrive(&hready);
                }
                bst[3] += tcd_clock() - tb;
            }
            if (next && kn < 128) {  // short instances: finish the doublings
                for (; kn < 128; kn <<= 1) newton_step(bpB, hsn, partB, tmpB, bt, F, kn, bsync);
                if (bt == 0) tc::mbar_arrive(&hready);
            }
        }
        if (blockIdx.x == 0 && bt == 0) {
            tcd_stats[8] = bst[0];
            tcd_stats[9] = bst[1];
            tcd_stats[11] = bst[3];
        }
    } else if (warp == (TCD_T + TCD_BLD) / 32) {
        // ---- warp 11, one lane: tile K's 16 UMMAs once the builders have written it
        //      and the compute warps have read block K+1 of the planes (tile K must
        //      not land before that read).  The issue blocks while the tensor core's
        //      queue is full (~1.8k cycles per tile), which is why it is not a
        //      builder lane: the builders' Newton steps and next tile would wait. ----
        if (lane == 0) {
            constexpr uint32_t ID_E = tc::idesc_u8(128, BROWS_E), ID_O = tc::idesc_u8(128, BROWS_O);
            uint32_t fph[2] = {0, 0}, bph[2] = {0, 0};
            uint32_t T = 0;
            long long mst[3] = {0, 0, 0};
            for (int64_t inst = blockIdx.x; inst < g.count; inst += gridDim.x)
                for (int K = 0; K <= Kq; ++K, ++T) {
                    const int b = T & 1;
                    long long tb = tcd_clock();
                    tc::mbar_wait(&built[b], bph[b]);
                    bph[b] ^= 1;
                    mst[0] += tcd_clock() - tb;
                    tb = tcd_clock();
                    tc::mbar_wait(&full[b], fph[b]);
                    fph[b] ^= 1;
                    if (TCD_STATS) {
                        const long long tn = clock64();
                        mst[1] += tn - tb;          // waited for the planes' read
                        mst[2] += tn - full_ts[b];  // its arrive -> seen here
                    }
                    tc::fence_after_sync();
                    const uint32_t hb = tc::smem_u32(sH + b * HBUF);
                    const bool odd = K & 1;
                    const uint32_t bb = tc::smem_u32(sBE) - (odd ? 128u : 0u);
                    const uint32_t idesc = odd ? ID_O : ID_E;
                    const uint32_t col = uint32_t(K & ~1);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            tc::mma_u8(tbase + 64 * u + col, tc::desc_sw128(hb + u * TILE + 32 * k),
                                       tc::desc_sw128(bb + 32 * k), idesc, 1u);
                    tc::commit(&empty[b]);
                    issue_ts[b] = tcd_clock();
                }
            if (blockIdx.x == 0) {
                tcd_stats[10] = mst[0];
                tcd_stats[14] = mst[1];
                tcd_stats[15] = mst[2];
            }
        }
        __syncwarp();
    } else {
        uint32_t eph[2] = {0, 0}, hph = 0;
        int pend[2] = {0, 0};
        int ip = 0;
        uint32_t T = 0;
        auto free_buf = [&](int b) {  // the tile handed off in buffer b is done
            if (pend[b]) {
                tc::mbar_wait(&empty[b], eph[b]);
                eph[b] ^= 1;
                --pend[b];
            }
        };
        auto bar = [] { asm volatile("bar.sync 1, 256;" ::: "memory"); };
        const uint32_t lane_addr = tbase + (uint32_t(32 * (warp & 3)) << 16);
        long long st[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int64_t inst = blockIdx.x; inst < g.count; inst += gridDim.x, ++ip) {
            const uint32_t* a = g.A + inst * g.lda;
            const uint32_t* b = g.B + inst * g.ldb;
            long long tp = tcd_clock();
            // ---- B' operand (rows 64 v + j), B'[0..256), zero TMEM, S_0 = 0 ----
            for (int u = tid; u < mB * 8; u += TCD_T) {
                const int j = u >> 3, c = u & 7;
                uint32_t wv[16];
                {  // B'[k] = b[nb - 1 - k], k = 128 j + 16 c + t: 16 words of b read backwards
                    const int k0 = 128 * j + 16 * c;
                    uint32_t rv[16];
                    if (k0 + 16 <= nb) {
                        load16(b + (nb - 16 - k0), 16, rv);
#pragma unroll
                        for (int t = 0; t < 16; ++t) wv[t] = rv[15 - t];
                    } else {
#pragma unroll
                        for (int t = 0; t < 16; ++t) wv[t] = k0 + t < nb ? __ldg(b + (nb - 1 - k0 - t)) : 0u;
                    }
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
            bp01[tid] = tid < nb ? __ldg(b + (nb - 1 - tid)) : 0u;
            bnc[tid] = (tid < 128 && 128 + tid < nb) ? __ldg(b + (nb - 129 - tid)) : 0u;
            if (tid < 128) {
                sS[tid] = 0;
                qz[tid] = 0;  // Q block 0 (a previous instance's values)
            }
            uint32_t aK = (tid < 128 && tid < na) ? __ldg(a + (na - 1 - tid)) : 0u;  // A' block 0
            if (warp < 4) {
#pragma unroll
                for (int c0 = 0; c0 < 512; c0 += 32) tmem_st32_zero(lane_addr + c0);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            bar();
            st[0] += tcd_clock() - tp;
            tp = tcd_clock();
            // ---- h = B'^-1 mod X^128: computed by the builder warps ----
            tc::mbar_wait(&hready, hph);
            hph ^= 1;
            const uint32_t* hs = hsp + 256 * (ip & 1) + 128;
            st[1] += tcd_clock() - tp;
            tp = tcd_clock();

            // ---- the step matrix M = T_h T_B1 (see the header), negated, into registers ----
            // u[r] = M[r][0] = sum_{t <= r} h[r - t] B'[128 + t]
            // (FAST: M is kept in Montgomery form, M 2^32 mod p, so that each entry and
            // each phase-A partial costs one REDC: the walk runs on B' 2^64 mod p)
            toeplitz_partials<FAST>(hs, bnc, 128, 128, part, F);
            uint32_t* bw = sE;  // B'[k] (2^64 mod p when FAST), k < 128
            if (tid < 128) bw[tid] = FAST ? reduce_odd(uint64_t(bp01[tid]) * F.r2, F) : bp01[tid];
            bar();
            if (tid < 128) {
                const uint32_t u = partials_sum<FAST>(part, 128, 128, tid, F);
                tmp[tid] = FAST ? reduce_odd(uint64_t(u) * F.r2, F) : u;
            }
            bar();
            {
                // diagonal r - m = dl of M, walked from its first entry with
                // M[r][m] = M[r-1][m-1] + h[r] B'[128 - m]; stored as p - M, rows of 128
                // words, word groups of 4 XOR-swizzled by the row group (conflict-free
                // 16-byte reads below)
                uint32_t* Mst = reinterpret_cast<uint32_t*>(sH);
                const int dl = tid - 127;
                if (dl < 128) {
                    int r = dl >= 0 ? dl : 0, m = dl >= 0 ? 0 : -dl;
                    uint64_t acc = dl >= 0 ? uint64_t(tmp[dl]) : uint64_t(hs[0]) * bw[128 + dl];
                    auto out = [&](uint64_t x) {
                        return negmod(FAST ? redc(fold(x, F), F) : reduce(x, F), F);
                    };
                    auto at = [](int r, int m) { return r * 128 + (m ^ (((r >> 2) & 7) << 2)); };
                    Mst[at(r, m)] = out(acc);
                    const int len = 128 - (dl >= 0 ? dl : -dl);  // entries on this diagonal
                    int i = 1;
                    if (FAST) {  // fold_terms >= 16: fold, 16 terms, fold, ... (pipelined)
                        acc = fold(acc, F);
                        for (; i + 16 <= len; i += 16) {
#pragma unroll
                            for (int q = 0; q < 16; ++q) {
                                acc = mad_wide(hs[r + i + q], bw[128 - (m + i + q)], acc);
                                Mst[at(r + i + q, m + i + q)] = out(acc);
                            }
                            acc = fold(acc, F);
                        }
                    }
                    uint32_t since = 1;
                    for (; i < len; ++i) {
                        if (++since > F.fold_terms) {
                            acc = fold(acc, F);
                            since = 1;
                        }
                        acc = mad_wide(hs[r + i], bw[128 - (m + i)], acc);
                        Mst[at(r + i, m + i)] = out(acc);
                    }
                }
            }
            bar();
            // thread (row group gq: rows 4 gq..4 gq+3, term part pq: terms 16 pq..16 pq+15)
            const int gq = tid & 31, pq = tid >> 5;
            const bool upper = pq > (gq >> 2);  // block (rows 4gq.., terms 16pq..) above the diagonal
            const int qx = (pq >> 1) & 3;       // slot swizzle of Q's words 16 pq .. 16 pq + 15
            // the diagonal blocks' strictly upper halves of U (phase A): thread = (row dr,
            // half dh of the block's 16 terms), window xw[j] = X[dr - (dt0 + j)]
            const int dr = tid >> 1, dh = tid & 1, dt0 = 16 * (dr >> 4) + 8 * dh;
            uint32_t mneg[4][16], hw[19], xw[8];
            {
                const uint32_t* Mst = reinterpret_cast<const uint32_t*>(sH);
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const uint4 v = *reinterpret_cast<const uint4*>(
                            Mst + (4 * gq + k) * 128 + ((16 * pq + 4 * jj) ^ ((gq & 7) << 2)));
                        mneg[k][4 * jj] = v.x;
                        mneg[k][4 * jj + 1] = v.y;
                        mneg[k][4 * jj + 2] = v.z;
                        mneg[k][4 * jj + 3] = v.w;
                    }
                // this thread's Toeplitz window for the merged phase B (see step K):
                // lower and diagonal blocks take h (zeros before it), strictly upper
                // blocks X[j] = B'[256 + j] for j < 0, zero for j >= 0 (bnc + 128)
                const uint32_t* wsrc = upper ? bnc + 128 : hs;
#pragma unroll
                for (int i = 0; i < 19; ++i) hw[i] = wsrc[4 * gq - 16 * pq - 15 + i];
#pragma unroll
                for (int j = 0; j < 8; ++j) xw[j] = bnc[128 + dr - dt0 - j];
            }
            if (tid < 128) {  // Z_0 = A'_0 (no planes, no corrections yet)
                sS[tid] = aK;
                const int kn = 128 + tid;  // prefetch A' block 1
                aK = kn < na ? __ldg(a + (na - 1 - kn)) : 0u;
            }
            bar();  // M read (the builders reuse the H buffers), Z_0 in place
            st[3] += tcd_clock() - tp;

            // Step K: Q_K = T_h Z_K - M Q_{K-1} with Z_K = A'_K - S_K - L_K in sS (the
            // planes hold tiles <= K-2, L_K = Q_{K-2}'s terms outside them, from the
            // compute warps' upper-block threads in phase B).  -M Q_{K-1} (phase A) is
            // formed as soon as Q_{K-1} is out, T_h Z_K and U Q_{K-1} (phase B) once S_K
            // has been read: 64 MACs per thread each.
            uint32_t pm[4] = {0, 0, 0, 0};  // this thread's partials of -M Q_{K-1}
            const uint32_t ft = F.fold_terms;
            for (int K = 0; K < Kq; ++K, ++T) {
                uint32_t* qk = qz + 128 * K;  // Q block K
                {
                    TCD_T0();
                    // T_h is lower triangular and L's matrix strictly upper: a thread whose
                    // block lies above the diagonal has no T_h Z_K terms and forms its
                    // part of L_{K+1} = U Q_{K-1} instead (same instruction stream, its
                    // window holds B' and its vector is Q_{K-1}); the diagonal blocks'
                    // L halves come from the previous step's phase A.
                    const uint32_t* vsrc = upper ? qk - 128 : sS;
                    uint32_t z[16];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint4 zv = *reinterpret_cast<const uint4*>(vsrc + 16 * pq + 4 * (i ^ (upper ? qx : 0)));
                        z[4 * i] = zv.x; z[4 * i + 1] = zv.y; z[4 * i + 2] = zv.z; z[4 * i + 3] = zv.w;
                    }
                    uint64_t a1[4] = {0, 0, 0, 0};
#ifndef TCD_NOMV
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            a1[k] = mad_wide(hw[k - j + 15], z[j], a1[k]);  // h[4gq + k - (16pq + j)]
                            if (!FAST && ft < 4) a1[k] = fold(a1[k], F);
                        }
                        if (!FAST && ft >= 4 && ft < 16 && (j & 3) == 3)
#pragma unroll
                            for (int k = 0; k < 4; ++k) a1[k] = fold(a1[k], F);
                    }
#endif
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t rk = reduce_t<FAST>(a1[k], F);
                        part[pq * 128 + 4 * gq + k] = (upper ? 0u : rk) + pm[k];
                        if (upper) partL[pq * 128 + 4 * gq + k] = rk;
                    }
                    bar();
                    TCD_ACC(6);
                }
                {
                    TCD_T0();
                    if (tid < 128) {
                        const int k1 = 128 * K + tid;
                        const uint32_t v1 = k1 < mu ? partials_sum<FAST>(part, 128, 128, tid, F) : 0u;
                        qk[swz_word(tid)] = v1;  // Q is stored slot-swizzled (tctile.cuh, build_unit)
                        if (k1 < mu) fan_store<FAN>(g.Q, inst * g.ldq + (mu - 1 - k1), v1);
                    } else {
                        qk[tid] = 0;  // Q block K+1: zero until solved (the last tile reads it)
                        if (K >= 1 && K + 1 < Kq) {  // L_{K+1} = U Q_{K-1}, row i
                            const int i = tid - 128, pd = i >> 4;
                            uint64_t v = partL[i];  // the diagonal block's part (step K-1's phase A)
#pragma unroll
                            for (int p = 1; p < 8; ++p) v += p > pd ? partL[p * 128 + i] : 0u;  // blocks above
                            lateb[i] = reduce_t<FAST>(v, F);
                        }
                    }
                    bar();
                    if (tid == 0) tc::mbar_arrive(&qready[T & 1]);  // the builders take tile K
                    TCD_ACC(4);
                }
                if (K + 1 < Kq) {  // phase A of step K+1: -M Q_K
                    TCD_T0();
                    uint32_t q[16];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint4 qv = *reinterpret_cast<const uint4*>(qk + 16 * pq + 4 * (i ^ qx));
                        q[4 * i] = qv.x; q[4 * i + 1] = qv.y; q[4 * i + 2] = qv.z; q[4 * i + 3] = qv.w;
                    }
                    uint64_t a2[4] = {0, 0, 0, 0};
                    // the diagonal blocks of U Q_K (L_{K+2}), 8 terms per thread
                    uint64_t ad = 0;
                    {
                        const uint4 d0 = *reinterpret_cast<const uint4*>(qk + swz_word(dt0));
                        const uint4 d1 = *reinterpret_cast<const uint4*>(qk + swz_word(dt0 + 4));
                        const uint32_t dq[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            ad = mad_wide(xw[j], dq[j], ad);
                            if (!FAST && ft < 8) ad = fold(ad, F);
                        }
                    }
#ifndef TCD_NOMV
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            a2[k] = mad_wide(mneg[k][j], q[j], a2[k]);
                            if (!FAST && ft < 4) a2[k] = fold(a2[k], F);
                        }
                        if (!FAST && ft >= 4 && ft < 16 && (j & 3) == 3)
#pragma unroll
                            for (int k = 0; k < 4; ++k) a2[k] = fold(a2[k], F);
                    }
#endif
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        pm[k] = FAST ? redc(fold(a2[k], F), F) : reduce(a2[k], F);  // M: Montgomery
                    {
                        uint32_t dv = reduce_t<FAST>(ad, F);
                        dv += __shfl_xor_sync(0xffffffffu, dv, 1);  // the row's two halves (< 2p)
                        if (!dh) partL[dr] = dv;
                    }
                    TCD_ACC(7);
                }
                {
                    TCD_T0();
                    // Z_{K+1} = A'_{K+1} - S_{K+1} - L_{K+1}: S from the planes once tile
                    // K-1 is done (block K+1 then holds tiles <= K-1)
                    // (tile K-1 is waited for at every step, the last one too: a
                    // parity wait must never fall two phases behind its mbarrier)
                    {
                        const long long tw = tcd_clock();
                        free_buf((T + 1) & 1);
                        const long long te = tcd_clock();
                        st[9] += te - tw;                              // waited for tile K-1
                        if (K > 0) st[10] += te - issue_ts[(T + 1) & 1];  // its issue -> seen done
                    }
                    // warp 11 may issue tile K as soon as block K+1 is in registers (the
                    // planes' rows of warps 0-3): full[] counts those four warps, so the
                    // tensor core restarts while Z_{K+1} is still being formed
                    auto release_tile = [&] {
                        tc::fence_before_sync();
                        __syncwarp();
                        if (lane == 0) {
                            if (TCD_STATS && tid == 0) full_ts[T & 1] = clock64();
                            tc::mbar_arrive(&full[T & 1]);
                        }
                    };
                    if (K + 1 < Kq) {
                        tc::fence_after_sync();
                        if (warp < 4) {
                            uint32_t x[7];
#pragma unroll
                            for (int s = 0; s < 7; ++s) x[s] = tmem_ld1(lane_addr + 64 * s + K + 1);
                            tc::tmem_ld_wait();
                            release_tile();
                            uint32_t zz = submod(aK, combine_planes(x, g.c_hi, F), F);
                            if (K + 1 >= 2) zz = submod(zz, lateb[tid], F);
                            sS[tid] = zz;
                            const int kn = 128 * (K + 2) + tid;  // prefetch A' block K+2
                            aK = kn < na ? __ldg(a + (na - 1 - kn)) : 0u;
                        }
                        tc::fence_before_sync();
                    } else if (warp < 4) {
                        release_tile();
                    }
                    bar();
                    ++pend[T & 1];
                    TCD_ACC(2);
                }
            }
            long long tq = tcd_clock();
            // ---- the last tile (Q_{Kq-1}'s upper triangle), then the remainder ----
            if (tid == 0) {
                if (TCD_STATS) full_ts[T & 1] = clock64();
                tc::mbar_arrive(&qready[T & 1]);
            }
            if (warp < 4 && lane == 0) tc::mbar_arrive(&full[T & 1]);
            ++pend[T & 1];
            ++T;
            // r[na-1-k] = A'[k] - (Q B')[k], k in [mu, na): 8 blocks per TMEM load, the
            // dividend words loaded while the last tiles run (blocks < 64: <= 4 rounds)
            {
                const int r = 32 * (warp & 3) + lane;
                const int cfirst = mu >> 7, clast = (na - 1) >> 7;
                const int64_t rb = inst * g.ldr;
                uint32_t av[4][8];
#pragma unroll
                for (int it = 0; it < 4; ++it)
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int k = 128 * (cfirst + 8 * (warp >> 2) + 16 * it + e) + r;
                        av[it][e] = (k >= mu && k < na) ? __ldg(a + (na - 1 - k)) : 0u;
                    }
                free_buf(0);
                free_buf(1);
                tc::fence_after_sync();
#pragma unroll
                for (int it = 0; it < 4; ++it) {
                    const int c0 = cfirst + 8 * (warp >> 2) + 16 * it;
                    if (c0 > clast) break;
                    uint32_t x[7][8];
#pragma unroll
                    for (int s = 0; s < 7; ++s) tmem_ld8(lane_addr + 64 * s + c0, x[s]);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int k = 128 * (c0 + e) + r;
                        if (k >= mu && k < na) {
                            const uint32_t xs[7] = {x[0][e], x[1][e], x[2][e], x[3][e], x[4][e],
                                                    x[5][e], x[6][e]};
                            fan_store<FAN>(g.R, rb + (na - 1 - k),
                                           submod(av[it][e], combine_planes(xs, g.c_hi, F), F));
                        }
                    }
                }
            }
            tc::fence_before_sync();
            bar();  // TMEM read before the next instance zeroes it
            tc::fence_after_sync();
            st[5] += tcd_clock() - tq;
        }
        if (blockIdx.x == 0 && tid == 0)
            for (int i = 0; i < 8; ++i) tcd_stats[i] = st[i];
        if (blockIdx.x == 0 && tid == 0) {
            tcd_stats[12] = st[9];
            tcd_stats[13] = st[10];
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) tc::tmem_free<512>(tbase);
}

}  // namespace

bool tcdiv_supported(int64_t na, int64_t nb, int64_t count, int64_t s) {
    const bool fits = nb >= 2 && na >= nb && na <= TCD_MAXA && nb <= TCM_MAXN;
    return tc_route("MMM_DIV_TC", s, fits,
                    nb >= 512 && na - nb + 1 >= 512 &&
                        double(na - nb + 1) * double(nb) * double(count) >= 1.0e9);
}

void launch_tcdiv_batched(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                          const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, Fan Q,
                          int64_t ldq, Fan R, int64_t ldr, cudaStream_t st) {
    if (count <= 0) return;
    if (!(nb >= 2 && na >= nb && na <= TCD_MAXA && nb <= TCM_MAXN))
        throw Error(ST_INVALID, "tensor-core division: needs 2 <= nb <= 4096, nb <= na <= 8192");
    TcDivArgs g{};
    g.A = A;
    g.B = B;
    g.lda = lda;
    g.ldb = ldb;
    g.ldq = ldq;
    g.ldr = ldr;
    g.na = int(na);
    g.nb = int(nb);
    g.count = count;
    g.Q = Q;
    g.R = R;
    g.Fp = F;
    for (int s = 0; s < 3; ++s) {
        uint64_t x = 1;
        for (int e = 0; e < 32 + 8 * s; ++e) x = (x * 2) % F.p;
        g.c_hi[s] = uint32_t(x);
    }
    const bool fan = Q.n > 1 || R.n > 1, fast = F.odd && F.fold_terms >= 16;
    auto kern = fan ? (fast ? tcdiv_kernel<true, true> : tcdiv_kernel<true, false>)
                    : (fast ? tcdiv_kernel<false, true> : tcdiv_kernel<false, false>);
    MMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(D_SMEM_BYTES)));
    const int blocks = int(std::min<int64_t>(count, sm_count()));
    kern<<<blocks, TCD_ALL, D_SMEM_BYTES, st>>>(g);
    check_launch("tcdiv_kernel", dim3(blocks), dim3(TCD_ALL));
    if (getenv("MMM_TC_STATS")) {
        long long h[16];
        MMM_CUDA(cudaMemcpyFromSymbolAsync(h, tcd_stats, sizeof(h), 0, cudaMemcpyDeviceToHost, st));
        MMM_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "tcdiv stats (CTA 0, thread 0): prologue=%lld h_wait=%lld tmem+Z=%lld "
                "M=%lld Qsum=%lld tail=%lld MV_B=%lld MV_A=%lld cycles | builders: wait_q=%lld build=%lld (issuer: wait_built=%lld) newton=%lld | mma_wait=%lld issue_to_done=%lld | issuer: full_wait=%lld full_arrive_to_seen=%lld\n",
                h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9], h[10], h[11], h[12], h[13], h[14], h[15]);
    }
}

}  // namespace mmm_cu
