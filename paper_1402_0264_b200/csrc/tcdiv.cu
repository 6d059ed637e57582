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
// tcmul.cu with Q on the Toeplitz side: after step K the tensor core adds
// tile H_K (built from Q_K and Q_{K-1}) times all of B' into the seven TMEM
// limb planes.  Step K+1 reads block K+1 of that sum back from TMEM (one
// column per plane), adds the part of tile H_{K+1} that Q_K already
// determines (its upper triangle against B'_0, on the CUDA cores), and solves
// the 128 x 128 triangular system for Q_{K+1} (the CUDA cores again).  After
// the last block one more tile completes Q B' and the remainder comes out of
// TMEM in one pass.  Shapes: na <= 8192, nb <= 4096 (cfg5: 8192 / 4096 terms).
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

constexpr int TCD_T = 256;
constexpr int TCD_MAXA = 8192;
constexpr int TCD_QWORDS = TCM_APAD + TCD_MAXA + 256;  // Q, padded like a_pad
// shared layout (bytes, 1024-aligned base)
constexpr uint32_t D_OFF_H = 0;                           // one H buffer (4 limb tiles)
constexpr uint32_t D_OFF_BE = D_OFF_H + HBUF;
constexpr uint32_t D_OFF_BO = D_OFF_BE + BROWS_E * 128;
constexpr uint32_t D_OFF_Q = D_OFF_BO + BROWS_O * 128;    // u32 Q (padded)
constexpr uint32_t D_OFF_A = D_OFF_Q + TCD_QWORDS * 4;    // u32 a (as given)
constexpr uint32_t D_OFF_SM = D_OFF_A + TCD_MAXA * 4;     // small arrays
constexpr uint32_t D_SMALL = 128 + 256 + 128 + 128 + 1024 + 128;  // bp0, h (padded), S, E, parts, tmp
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
__device__ __forceinline__ void toeplitz_partials(const uint32_t* X, const uint32_t* W, int n,
                                                  int T, uint32_t* part, const FieldParams& F) {
    const int ng = n >> 2, np = T >> 4;
    const int tid = threadIdx.x;
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
                if (ft < 4) acc[k] = fold(acc[k], F);
            }
        }
        if (ft >= 4 && ft < 16)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] = fold(acc[k], F);
        cur[0] = nv.x;
        cur[1] = nv.y;
        cur[2] = nv.z;
        cur[3] = nv.w;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) part[p * n + r0 + k] = reduce(acc[k], F);
}

// y[i] = sum over the T/16 partials, mod p (threads i < n).
__device__ __forceinline__ uint32_t partials_sum(const uint32_t* part, int n, int T, int i,
                                                 const FieldParams& F) {
    uint64_t v = 0;
    for (int p = 0; p < (T >> 4); ++p) v += part[p * n + i];
    return reduce(v, F);
}

__device__ long long tcd_stats[8];
#define TCD_T0() const long long _t0 = clock64()
#define TCD_ACC(i) st[i] += clock64() - _t0

template <bool FAN>
__global__ void __launch_bounds__(TCD_T, 1) tcdiv_kernel(TcDivArgs g) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
    uint8_t* sH = sm + D_OFF_H;
    uint8_t* sBE = sm + D_OFF_BE;
    uint8_t* sBO = sm + D_OFF_BO;
    uint32_t* q_pad = reinterpret_cast<uint32_t*>(sm + D_OFF_Q);
    uint32_t* a_s = reinterpret_cast<uint32_t*>(sm + D_OFF_A);
    uint32_t* bp0 = reinterpret_cast<uint32_t*>(sm + D_OFF_SM);  // B'[0..128)
    uint32_t* hs = bp0 + 128 + 128;                               // B'^-1 mod X^128, 128 zeros before
    uint32_t* sS = hs + 128;                                      // block K of the sum
    uint32_t* sE = sS + 128;
    uint32_t* part = sE + 128;                                    // [8][128] partial sums
    uint32_t* tmp = part + 1024;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const FieldParams F = g.Fp;
    const int na = g.na, nb = g.nb;
    const int mu = na - nb + 1, db = nb - 1;
    const int mB = (nb + 127) >> 7;
    const int Kq = (mu + 127) >> 7;  // quotient blocks; tiles d = 0 .. Kq

    for (uint32_t i = tid; i < (BROWS_E + BROWS_O) * 128 / 16; i += TCD_T)
        reinterpret_cast<uint4*>(sBE)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < TCD_QWORDS; i += TCD_T) q_pad[i] = 0;
    for (int i = tid; i < 128; i += TCD_T) hs[i - 128] = 0;
    if (warp == 0) tc::tmem_alloc<512>(&tslot);
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = tslot;
    uint32_t ph = 0;
    constexpr uint32_t ID_E = tc::idesc_u8(128, BROWS_E), ID_O = tc::idesc_u8(128, BROWS_O);
    const uint32_t lane_addr = tbase + (uint32_t(32 * (warp & 3)) << 16);

    long long st[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t inst = blockIdx.x; inst < g.count; inst += gridDim.x) {
        const uint32_t* a = g.A + inst * g.lda;
        const uint32_t* b = g.B + inst * g.ldb;
        long long tp = clock64();
        // ---- stage a; B' operand copies (rows 64 v + j [+1]); B'_0; zero TMEM ----
        for (int i = tid; i < na; i += TCD_T) a_s[i] = __ldg(a + i);
        for (int u = tid; u < mB * 8; u += TCD_T) {
            const int j = u >> 3, c = u & 7;
            uint32_t wv[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const int k = 128 * j + 16 * c + t;  // B' index
                wv[t] = k < nb ? __ldg(b + (nb - 1 - k)) : 0u;
            }
            uint32_t L[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                limb_transpose(wv[4 * q], wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3], L[0][q],
                               L[1][q], L[2][q], L[3][q]);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                sts128(sBE, tc::sw128(64 * v + j, 16 * c), L[v][0], L[v][1], L[v][2], L[v][3]);
                sts128(sBO, tc::sw128(64 * v + j + 1, 16 * c), L[v][0], L[v][1], L[v][2], L[v][3]);
            }
        }
        if (tid < 128) bp0[tid] = tid < nb ? __ldg(b + (nb - 1 - tid)) : 0u;
        if (warp < 4) {
#pragma unroll
            for (int c0 = 0; c0 < 512; c0 += 32) tmem_st32_zero(lane_addr + c0);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        __syncthreads();
        st[0] += clock64() - tp;
        tp = clock64();
        // ---- h = B'^-1 mod X^128 by Newton doubling ----
        if (tid == 0) hs[0] = invmod(bp0[0], F);
        __syncthreads();
        for (int k = 1; k < 16; k <<= 1) {
            // e[i] = sum_{m<k} B'[k+i-m] h[m]  (i < k): coefficients [k, 2k) of B' h_k
            if (tid < k) {
                Acc e;
                for (int m = 0; m < k; ++m) e.add(bp0[k + tid - m], hs[m], F);
                tmp[tid] = reduce(e.v, F);
            }
            __syncthreads();
            if (tid < k) {  // h[k+i] = -sum_{m<=i} h[i-m] e[m]
                Acc s;
                for (int m = 0; m <= tid; ++m) s.add(hs[tid - m], tmp[m], F);
                hs[k + tid] = negmod(reduce(s.v, F), F);
            }
            __syncthreads();
        }
        for (int k = 16; k < 128; k <<= 1) {  // the same doubling with sliding products
            toeplitz_partials(bp0 + k, hs, k, k, part, F);
            __syncthreads();
            if (tid < k) tmp[tid] = partials_sum(part, k, k, tid, F);
            __syncthreads();
            toeplitz_partials(hs, tmp, k, k, part, F);  // h[i-m], zero for i < m
            __syncthreads();
            if (tid < k) hs[k + tid] = negmod(partials_sum(part, k, k, tid, F), F);
            __syncthreads();
        }

        st[1] += clock64() - tp;
        for (int K = 0; K <= Kq; ++K) {
            if (K >= 1) {
                TCD_T0();
                tc::mbar_wait(&mbar, ph);  // tile K-1 is in the planes
                ph ^= 1;
                tc::fence_after_sync();
                TCD_ACC(2);
            }
            if (K < Kq) {
                TCD_T0();
                // ---- block K of the running sum, from TMEM (warps 0-3: row = lane);
                //      block K of Q cleared (U below reads it as zeros) ----
                uint32_t* qk = q_pad + TCM_APAD + 128 * K;
                if (warp < 4) {
                    uint32_t x[7];
#pragma unroll
                    for (int s = 0; s < 7; ++s) x[s] = tmem_ld1(lane_addr + 64 * s + K);
                    tc::tmem_ld_wait();
                    sS[32 * warp + lane] = combine_planes(x, g.c_hi, F);
                } else {
                    qk[tid - 128] = 0;
                }
                __syncthreads();
                // ---- U = (upper triangle of H_K) B'_0: the part of block K that
                //      Q_{K-1} determines beyond the planes; E = A' - S - U ----
                toeplitz_partials(qk, bp0, 128, 128, part, F);
                __syncthreads();
                if (tid < 128) {
                    const int k1 = 128 * K + tid;
                    const uint32_t a1 = k1 < na ? a_s[na - 1 - k1] : 0u;
                    sE[tid] = submod(submod(a1, sS[tid], F), partials_sum(part, 128, 128, tid, F), F);
                }
                __syncthreads();
                // ---- Q_K = E * h mod X^128 ----
                toeplitz_partials(hs, sE, 128, 128, part, F);
                __syncthreads();
                if (tid < 128) {
                    const int k1 = 128 * K + tid;
                    const uint32_t v1 = k1 < mu ? partials_sum(part, 128, 128, tid, F) : 0u;
                    qk[tid] = v1;
                    if (k1 < mu) fan_store<FAN>(g.Q, inst * g.ldq + (mu - 1 - k1), v1);
                }
                __syncthreads();
                TCD_ACC(3);
            }
            // ---- tile H_K (Q_K lower, Q_{K-1} upper) into the planes ----
            {
            TCD_T0();
            build_h(sH, q_pad, K);
            tc::fence_async_smem();
            tc::fence_before_sync();
            __syncthreads();
            tc::fence_after_sync();
            TCD_ACC(4);
            }
            if (tid == 0) {
                const uint32_t hb = tc::smem_u32(sH);
                const bool odd = K & 1;
                const uint32_t bb = tc::smem_u32(odd ? sBO : sBE);
                const uint32_t idesc = odd ? ID_O : ID_E;
                const uint32_t col = uint32_t(K & ~1);
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        tc::mma_u8(tbase + 64 * u + col, tc::desc_sw128(hb + u * TILE + 32 * k),
                                   tc::desc_sw128(bb + 32 * k), idesc, 1u);
                tc::commit(&mbar);
            }
        }
        tp = clock64();
        tc::mbar_wait(&mbar, ph);  // the last tile
        ph ^= 1;
        tc::fence_after_sync();
        // ---- remainder: r[na-1-k] = A'[k] - (Q B')[k], k in [mu, na) ----
        {
            const int r = 32 * (warp & 3) + lane;
            const int cfirst = mu >> 7, clast = (na - 1) >> 7;
            const int64_t rb = inst * g.ldr;
            for (int c = cfirst + (warp >> 2); c <= clast; c += 2) {
                uint32_t x[7];
#pragma unroll
                for (int s = 0; s < 7; ++s) x[s] = tmem_ld1(lane_addr + 64 * s + c);
                tc::tmem_ld_wait();
                const int k = 128 * c + r;
                if (k >= mu && k < na) {
                    const uint32_t S = combine_planes(x, g.c_hi, F);
                    fan_store<FAN>(g.R, rb + (na - 1 - k), submod(a_s[na - 1 - k], S, F));
                }
            }
        }
        tc::fence_before_sync();
        __syncthreads();  // TMEM read before the next instance zeroes it
        tc::fence_after_sync();
        st[5] += clock64() - tp;
    }
    if (blockIdx.x == 0 && tid == 0)
        for (int i = 0; i < 8; ++i) tcd_stats[i] = st[i];
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tbase);
}

}  // namespace

bool tcdiv_supported(int64_t na, int64_t nb, int64_t count) {
    const bool fits = nb >= 2 && na >= nb && na <= TCD_MAXA && nb <= TCM_MAXN;
    if (const char* e = getenv("MMM_DIV_TC")) return atoi(e) != 0 && fits;
    return fits && nb >= 512 && na - nb + 1 >= 512 &&
           double(na - nb + 1) * double(nb) * double(count) >= 1.0e9;
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
    auto kern = (Q.n > 1 || R.n > 1) ? tcdiv_kernel<true> : tcdiv_kernel<false>;
    MMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(D_SMEM_BYTES)));
    const int blocks = int(std::min<int64_t>(count, sm_count()));
    kern<<<blocks, TCD_T, D_SMEM_BYTES, st>>>(g);
    check_launch("tcdiv_kernel", dim3(blocks), dim3(TCD_T));
    if (getenv("MMM_TC_STATS")) {
        long long h[8];
        MMM_CUDA(cudaMemcpyFromSymbolAsync(h, tcd_stats, sizeof(h), 0, cudaMemcpyDeviceToHost, st));
        MMM_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "tcdiv stats (CTA 0, thread 0): prologue=%lld newton=%lld mma_wait=%lld "
                "head_solve=%lld build=%lld tail=%lld cycles\n", h[0], h[1], h[2], h[3], h[4], h[5]);
    }
}

}  // namespace mmm_cu
