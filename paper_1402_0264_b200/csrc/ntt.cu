// ntt.cu -- NTT (number-theoretic FFT) multiplication over Z/pZ on sm_100a.
//
// New scope (the reference has no FFT; SPEC.md:385 lists FFT
// multiplication as a non-goal there).  Its parity anchor is uniqueness of
// the product: the result must equal oracle_mul (proj/src/oracle.cpp:8-15).
//
// Transform length N = 2^k >= na+nb-1 (needs 2^k | p-1), split N = N1*N2
// (four-step):
//   K1  column pass  : for each column n2, an N1-point transform over
//                      x[N2*n1 + n2] (zero-padded input), times w_N^(n2*k1);
//   K2  row pass     : per row k1, N2-point forward transforms of both
//                      operands, pointwise product, N2-point inverse,
//                      times w_N^-(n2*k1)     (fused: one read, one write);
//   K3  column pass  : inverse N1-point transforms, scaled by N^-1,
//                      written in natural order.
// Every sub-transform is a Stockham autosort network in shared memory
// (natural order in and out, ping-pong buffers) taking two radix-2 stages per
// pass in registers (stockham4: 189 -> 129 us for 2^21), twiddles staged in
// shared memory with Shoup companions w' = floor(w * 2^32 / p), so each
// butterfly is add/sub + one Shoup product (IMAD.HI + 2 IMAD + correction).
// Between passes the data stays in an N-word workspace per operand (L2).
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace mmm_cu {

namespace {

constexpr int NTT_T = 256;
constexpr int NTT_PHASE_COLS = 4;  // column granularity of the sharded phases

__device__ __forceinline__ uint32_t shoup(uint32_t x, uint32_t w, uint32_t wp, uint32_t p) {
    const uint32_t q = __umulhi(x, wp);
    const uint32_t r = x * w - q * p;
    return r >= p ? r - p : r;
}
__device__ __forceinline__ uint32_t add_p(uint32_t a, uint32_t b, uint32_t p) {
    const uint32_t s = a + b;
    return s >= p ? s - p : s;
}
__device__ __forceinline__ uint32_t sub_p(uint32_t a, uint32_t b, uint32_t p) {
    return a >= b ? a - b : a + p - b;
}

// Butterfly halves, exact (LZ = false: canonical in and out) or lazy (LZ =
// true, p < 2^30: values in [0, 2p) in and out; Harvey's trick -- the sum
// needs one conditional subtraction of 2p, the difference none: a - b + 2p
// < 4p < 2^32 goes straight into a Shoup product, whose unreduced result
// x*w - q*p lies in [0, 2p) for any x < 2^32).  Half the ALU work per
// butterfly of the exact form, which the ALU-bound transform feels directly.
template <bool LZ>
__device__ __forceinline__ uint32_t bf_add(uint32_t a, uint32_t b, uint32_t p) {
    if (!LZ) return add_p(a, b, p);
    const uint32_t s = a + b, p2 = 2 * p;
    return s >= p2 ? s - p2 : s;
}
template <bool LZ>
__device__ __forceinline__ uint32_t shoup_l(uint32_t x, uint32_t w, uint32_t wp, uint32_t p) {
    if (!LZ) return shoup(x, w, wp, p);
    return x * w - __umulhi(x, wp) * p;
}
template <bool LZ>
__device__ __forceinline__ uint32_t bf_subw(uint32_t a, uint32_t b, uint2 w, uint32_t p) {
    return LZ ? shoup_l<true>(a - b + 2 * p, w.x, w.y, p) : shoup(sub_p(a, b, p), w.x, w.y, p);
}

// Device tables for one (p, N): roots of the two sub-transform lengths and
// the two-level four-step twiddles, each value followed by its Shoup
// companion (interleaved pairs).
struct NttPlan {
    uint32_t p;
    int logN, log1, log2;  // N = N1 * N2, N1 = 2^log1 (columns), N2 = 2^log2 (rows)
    uint32_t scale, scale_p;  // N^-1 mod p (+ companion)
    uint2* r1f;  // w_N1^j,  j < N1/2
    uint2* r1i;  // w_N1^-j
    uint2* r2f;  // w_N2^j,  j < N2/2
    uint2* r2i;
    uint2* tlo_f;  // w_N^e,  e < 2^LO
    uint2* thi_f;  // w_N^(e << LO), e < N >> LO
    uint2* tlo_i;
    uint2* thi_i;
};
constexpr int LO = 10;

// Shared-memory data words are stored padded, one word per 32: the Stockham
// passes write at strides 8 and 64 (radix-8), which without padding hit 4-8
// words per bank (ncu: ~47 % of ntt_rows' shared wavefronts were replays).
__device__ __forceinline__ int PD(int i) { return i + (i >> 5); }
constexpr int padded_words(int n) { return n + (n >> 5) + 1; }

// Two Stockham stages at once (radix-4 step): the unit (q, pp), pp < H/2 with
// H = half/sp, reads the four words x[q + sp*(pp + j*H/2)], j < 4, runs the
// stage-s butterflies (pp, pp + H/2) and the stage-(s+1) butterflies on their
// outputs in registers, and writes y[q + sp*(4pp + b0 + 2*b1)]: half the
// passes, barriers and index arithmetic of two radix-2 stages.
template <bool LZ>
__device__ uint32_t* stockham4(uint32_t* x, uint32_t* y, int logL, int logc, const uint2* tw,
                               uint32_t p) {
    const int L = 1 << logL, half = L >> 1, cols = 1 << logc;
    int s = 0;
    // three stages per pass while at least three remain (radix-8 step): the
    // unit (q, pp), pp < H/4, owns x[q + sp*(pp + j*H/4)], j < 8; stage s
    // pairs (j, j+4), stage s+1 pairs (j, j+2) of the results, stage s+2 pairs
    // (0, 1); outputs land at y[q + sp*(8pp + b0 + 2 b1 + 4 b2)] (padded: PD).
    for (; s + 2 < logL && (logL - s) != 4; s += 3) {
        const int sp = 1 << s, Q = (half >> s) >> 2;
        for (int t = threadIdx.x; t < ((L >> 3) << logc); t += blockDim.x) {
            const int c = t & (cols - 1), u = t >> logc;
            const int pp = u >> s, q = u & (sp - 1);
            const int base = c + cols * q, st = cols * sp;
            uint32_t v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = x[PD(base + st * (pp + j * Q))];
            uint32_t e[8];  // e[2j + b0]: stage-s outputs of pair (j, j+4)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint2 w = tw[(pp + j * Q) * sp];
                e[2 * j] = bf_add<LZ>(v[j], v[j + 4], p);
                e[2 * j + 1] = bf_subw<LZ>(v[j], v[j + 4], w, p);
            }
            uint32_t f[8];  // f[4j + 2b1 + b0]... indexed f[j][b0][b1] = f[4j + 2 b0 + b1]
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint2 w = tw[(pp + j * Q) * 2 * sp];
#pragma unroll
                for (int b0 = 0; b0 < 2; ++b0) {
                    const uint32_t a0 = e[2 * j + b0], a1 = e[2 * (j + 2) + b0];
                    f[4 * j + 2 * b0] = bf_add<LZ>(a0, a1, p);
                    f[4 * j + 2 * b0 + 1] = bf_subw<LZ>(a0, a1, w, p);
                }
            }
            const uint2 w = tw[pp * 4 * sp];
#pragma unroll
            for (int b0 = 0; b0 < 2; ++b0)
#pragma unroll
                for (int b1 = 0; b1 < 2; ++b1) {
                    const uint32_t a0 = f[2 * b0 + b1], a1 = f[4 + 2 * b0 + b1];
                    const int o = 8 * pp + b0 + 2 * b1;
                    y[PD(base + st * o)] = bf_add<LZ>(a0, a1, p);
                    y[PD(base + st * (o + 4))] = bf_subw<LZ>(a0, a1, w, p);
                }
        }
        __syncthreads();
        uint32_t* t = x;
        x = y;
        y = t;
    }
    for (; s + 1 < logL; s += 2) {
        const int sp = 1 << s, H = half >> s, H2 = H >> 1;
        for (int t = threadIdx.x; t < ((L >> 2) << logc); t += blockDim.x) {
            const int c = t & (cols - 1), u = t >> logc;
            const int pp = u >> s, q = u & (sp - 1);  // u = q + sp*pp, pp < H/2
            const int base = c + cols * q, st = cols * sp;
            const uint32_t a0 = x[PD(base + st * pp)];
            const uint32_t a1 = x[PD(base + st * (pp + H2))];
            const uint32_t a2 = x[PD(base + st * (pp + H))];
            const uint32_t a3 = x[PD(base + st * (pp + H2 + H))];
            const uint2 w0 = tw[pp * sp], w1 = tw[(pp + H2) * sp], w2 = tw[pp * 2 * sp];
            // stage s: (a0, a2) -> y[2pp], y[2pp+1]; (a1, a3) -> y[2pp+H], y[2pp+H+1]
            const uint32_t e0 = bf_add<LZ>(a0, a2, p), e1 = bf_subw<LZ>(a0, a2, w0, p);
            const uint32_t f0 = bf_add<LZ>(a1, a3, p), f1 = bf_subw<LZ>(a1, a3, w1, p);
            // stage s+1, q' = q + sp*b0: (e_b0, f_b0) -> y'[4pp + b0], y'[4pp + b0 + 2]
            y[PD(base + st * (4 * pp))] = bf_add<LZ>(e0, f0, p);
            y[PD(base + st * (4 * pp + 2))] = bf_subw<LZ>(e0, f0, w2, p);
            y[PD(base + st * (4 * pp + 1))] = bf_add<LZ>(e1, f1, p);
            y[PD(base + st * (4 * pp + 3))] = bf_subw<LZ>(e1, f1, w2, p);
        }
        __syncthreads();
        uint32_t* t = x;
        x = y;
        y = t;
    }
    if (s < logL) {  // odd logL: one radix-2 stage left
        const int sp = 1 << s;
        for (int t = threadIdx.x; t < (half << logc); t += blockDim.x) {
            const int c = t & (cols - 1), i = t >> logc;
            const int pp = i >> s, q = i & (sp - 1);
            const uint32_t a = x[PD(c + cols * (q + sp * pp))];
            const uint32_t b = x[PD(c + cols * (q + sp * (pp + half / sp)))];
            const uint2 w = tw[pp * sp];
            y[PD(c + cols * (q + sp * (2 * pp)))] = bf_add<LZ>(a, b, p);
            y[PD(c + cols * (q + sp * (2 * pp + 1)))] = bf_subw<LZ>(a, b, w, p);
        }
        __syncthreads();
        uint32_t* t = x;
        x = y;
        y = t;
    }
    return x;
}

template <bool LZ>
__device__ __forceinline__ uint32_t twiddle(uint32_t v, uint64_t e, const uint2* lo,
                                            const uint2* hi, uint32_t p) {
    const uint2 a = lo[e & ((1u << LO) - 1)];
    const uint2 b = hi[e >> LO];
    return shoup_l<LZ>(shoup_l<LZ>(v, a.x, a.y, p), b.x, b.y, p);
}

struct NttArgs {
    NttPlan P;
    const uint32_t* in[2];
    int64_t len[2], ld[2];
    uint32_t* work[2];  // N words per instance per operand
    uint32_t* out;
    int64_t nf, ldf;
    int cols;           // columns per CTA in the column passes
    int logc;           // log2(cols)
    int col0, row0;     // first column / row of this launch (sharded phases)
};

// K1: forward column transforms of both operands (grid.y = operand).
template <bool LZ>
__global__ void __launch_bounds__(NTT_T) ntt_cols_fwd(NttArgs g) {
    extern __shared__ __align__(16) uint32_t sm[];
    const NttPlan& P = g.P;
    const int N1 = 1 << P.log1, N2 = 1 << P.log2, C = g.cols;
    const int op = blockIdx.y;
    const int64_t inst = blockIdx.z;
    const uint32_t* in = g.in[op] + inst * g.ld[op];
    const int64_t len = g.len[op];
    uint32_t* work = g.work[op] + (inst << P.logN);
    uint2* tw = reinterpret_cast<uint2*>(sm);
    uint32_t* x = sm + N1;  // N1/2 uint2 = N1 words
    uint32_t* y = x + padded_words(C * N1);
    const int c0 = g.col0 + blockIdx.x * C;
    for (int j = threadIdx.x; j < N1 / 2; j += NTT_T) tw[j] = P.r1f[j];
    for (int t = threadIdx.x; t < C * N1; t += NTT_T) {
        const int c = t & (C - 1), n1 = t >> g.logc;
        const int64_t idx = int64_t(N2) * n1 + c0 + c;
        x[PD(t)] = idx < len ? in[idx] : 0u;
    }
    __syncthreads();
    uint32_t* r = stockham4<LZ>(x, y, P.log1, g.logc, tw, P.p);
    for (int t = threadIdx.x; t < C * N1; t += NTT_T) {
        const int c = t & (C - 1), k1 = t >> g.logc;
        const uint64_t e = uint64_t(c0 + c) * uint64_t(k1);
        work[int64_t(N2) * k1 + c0 + c] = twiddle<LZ>(r[PD(t)], e, P.tlo_f, P.thi_f, P.p);
    }
}

// K2: per row: forward both, pointwise product, inverse, inverse twiddle.
template <bool LZ>
__global__ void __launch_bounds__(NTT_T) ntt_rows(NttArgs g, FieldParams F) {
    extern __shared__ __align__(16) uint32_t sm[];
    const NttPlan& P = g.P;
    const int N2 = 1 << P.log2;
    const int k1 = g.row0 + blockIdx.x;
    const int64_t inst = blockIdx.z;
    uint32_t* wa = g.work[0] + (inst << P.logN) + int64_t(k1) * N2;
    const uint32_t* wb = g.work[1] + (inst << P.logN) + int64_t(k1) * N2;
    uint2* twf = reinterpret_cast<uint2*>(sm);
    uint2* twi = twf + N2 / 2;
    uint32_t* xa = sm + 2 * N2;
    uint32_t* ya = xa + padded_words(N2);
    uint32_t* xb = ya + padded_words(N2);
    uint32_t* yb = xb + padded_words(N2);
    for (int j = threadIdx.x; j < N2 / 2; j += NTT_T) {
        twf[j] = P.r2f[j];
        twi[j] = P.r2i[j];
    }
    for (int t = threadIdx.x; t < N2; t += NTT_T) {
        xa[PD(t)] = wa[t];
        xb[PD(t)] = wb[t];
    }
    __syncthreads();
    // the two forward transforms as one 2-column network: interleave? keep
    // them separate (same code, half the threads idle per stage otherwise)
    uint32_t* ra = stockham4<LZ>(xa, ya, P.log2, 0, twf, P.p);
    uint32_t* rb = stockham4<LZ>(xb, yb, P.log2, 0, twf, P.p);
    for (int t = threadIdx.x; t < N2; t += NTT_T) ra[PD(t)] = mulmod(ra[PD(t)], rb[PD(t)], F);
    __syncthreads();
    uint32_t* other = ra == xa ? ya : xa;
    uint32_t* rc = stockham4<LZ>(ra, other, P.log2, 0, twi, P.p);
    for (int t = threadIdx.x; t < N2; t += NTT_T) {
        const uint64_t e = (uint64_t(1) << P.logN) - (uint64_t(t) * uint64_t(k1));
        wa[t] = twiddle<LZ>(rc[PD(t)], e & ((uint64_t(1) << P.logN) - 1), P.tlo_f, P.thi_f, P.p);
    }
}

// K3: inverse column transforms, N^-1 scale, natural-order output.
template <bool LZ>
__global__ void __launch_bounds__(NTT_T) ntt_cols_inv(NttArgs g) {
    extern __shared__ __align__(16) uint32_t sm[];
    const NttPlan& P = g.P;
    const int N1 = 1 << P.log1, N2 = 1 << P.log2, C = g.cols;
    const int64_t inst = blockIdx.z;
    const uint32_t* work = g.work[0] + (inst << P.logN);
    uint32_t* out = g.out + inst * g.ldf;
    uint2* tw = reinterpret_cast<uint2*>(sm);
    uint32_t* x = sm + N1;
    uint32_t* y = x + padded_words(C * N1);
    const int c0 = g.col0 + blockIdx.x * C;
    for (int j = threadIdx.x; j < N1 / 2; j += NTT_T) tw[j] = P.r1i[j];
    for (int t = threadIdx.x; t < C * N1; t += NTT_T) {
        const int c = t & (C - 1), k1 = t >> g.logc;
        x[PD(t)] = work[int64_t(N2) * k1 + c0 + c];
    }
    __syncthreads();
    uint32_t* r = stockham4<LZ>(x, y, P.log1, g.logc, tw, P.p);
    for (int t = threadIdx.x; t < C * N1; t += NTT_T) {
        const int c = t & (C - 1), n1 = t >> g.logc;
        const int64_t idx = int64_t(N2) * n1 + c0 + c;
        if (idx < g.nf) out[idx] = shoup(r[PD(t)], P.scale, P.scale_p, P.p);
    }
}

// ------------------------------------------------------------ host side --
uint32_t pow_mod(uint64_t b, uint64_t e, uint32_t p) {
    uint64_t r = 1;
    b %= p;
    while (e) {
        if (e & 1) r = r * b % p;
        b = b * b % p;
        e >>= 1;
    }
    return uint32_t(r);
}

uint32_t primitive_root(uint32_t p) {
    std::vector<uint64_t> fac;
    uint64_t m = p - 1;
    for (uint64_t d = 2; d * d <= m; ++d)
        if (m % d == 0) {
            fac.push_back(d);
            while (m % d == 0) m /= d;
        }
    if (m > 1) fac.push_back(m);
    for (uint32_t gcand = 2; gcand < p; ++gcand) {
        bool ok = true;
        for (uint64_t q : fac)
            if (pow_mod(gcand, (p - 1) / q, p) == 1) {
                ok = false;
                break;
            }
        if (ok) return gcand;
    }
    return 1;
}

uint2 shoup_pair(uint32_t w, uint32_t p) {
    return make_uint2(w, uint32_t((uint64_t(w) << 32) / p));
}

std::vector<uint2> powers(uint32_t w, size_t n, uint32_t p) {
    std::vector<uint2> v(n);
    uint64_t x = 1;
    for (size_t j = 0; j < n; ++j) {
        v[j] = shoup_pair(uint32_t(x), p);
        x = x * w % p;
    }
    return v;
}

struct PlanCache {
    std::mutex mu;
    std::map<std::tuple<int, uint32_t, int>, std::unique_ptr<NttPlan>> plans;
} g_plans;

const NttPlan& get_plan(uint32_t p, int logN) {
    int dev = 0;
    MMM_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_plans.mu);
    auto key = std::make_tuple(dev, p, logN);
    auto it = g_plans.plans.find(key);
    if (it != g_plans.plans.end()) return *it->second;
    auto plan = std::make_unique<NttPlan>();
    NttPlan& P = *plan;
    P.p = p;
    P.logN = logN;
    P.log1 = logN / 2;
    P.log2 = logN - P.log1;
    const uint32_t g = primitive_root(p);
    const uint64_t N = uint64_t(1) << logN;
    const uint32_t wN = pow_mod(g, (p - 1) / N, p);
    const uint32_t wNi = pow_mod(wN, p - 2, p);
    const uint32_t w1 = pow_mod(wN, uint64_t(1) << P.log2, p);  // order N1
    const uint32_t w2 = pow_mod(wN, uint64_t(1) << P.log1, p);  // order N2
    const uint32_t ninv = pow_mod(uint32_t(N % p), p - 2, p);
    const uint2 sc = shoup_pair(ninv, p);
    P.scale = sc.x;
    P.scale_p = sc.y;
    auto upload = [](const std::vector<uint2>& v) {
        uint2* d = nullptr;
        MMM_CUDA(cudaMalloc(&d, std::max<size_t>(v.size(), 1) * sizeof(uint2)));
        MMM_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(uint2), cudaMemcpyHostToDevice));
        return d;
    };
    const size_t n1h = std::max<size_t>((size_t(1) << P.log1) / 2, 1);
    const size_t n2h = std::max<size_t>((size_t(1) << P.log2) / 2, 1);
    P.r1f = upload(powers(w1, n1h, p));
    P.r1i = upload(powers(pow_mod(w1, p - 2, p), n1h, p));
    P.r2f = upload(powers(w2, n2h, p));
    P.r2i = upload(powers(pow_mod(w2, p - 2, p), n2h, p));
    const size_t nlo = size_t(1) << LO, nhi = std::max<size_t>(N >> LO, 1);
    P.tlo_f = upload(powers(wN, nlo, p));
    P.thi_f = upload(powers(pow_mod(wN, nlo, p), nhi, p));
    P.tlo_i = upload(powers(wNi, nlo, p));
    P.thi_i = upload(powers(pow_mod(wNi, nlo, p), nhi, p));
    const NttPlan& ref = *plan;
    g_plans.plans.emplace(key, std::move(plan));
    return ref;
}

int log2_len(int64_t nf) {
    int k = 2;
    while ((int64_t(1) << k) < nf) ++k;
    return k;
}

template <bool LZ>
void run_ntt_launches(NttArgs g, const FieldParams& F, int N1, int N2, int64_t count,
                      int64_t chunk, const uint32_t* A, int64_t lda, const uint32_t* B,
                      int64_t ldb, uint32_t* Fo, int64_t ldf, size_t sm1, size_t sm2,
                      cudaStream_t st);

void run_ntt(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na, const uint32_t* B,
             int64_t ldb, int64_t nb, int64_t count, uint32_t* Fo, int64_t ldf, cudaStream_t st) {
    const int64_t nf = na + nb - 1;
    const int logN = log2_len(nf);
    if (logN > 30) throw Error(ST_INVALID, "ntt: product too long");
    const NttPlan& P = get_plan(F.p, logN);
    const int N1 = 1 << P.log1, N2 = 1 << P.log2;
    NttArgs g{};
    g.P = P;
    g.len[0] = na;
    g.len[1] = nb;
    g.nf = nf;
    // columns per CTA in the column passes: 4 for one large transform (more,
    // smaller CTAs: 111 vs 115 us at 2^21), 8 for batches (0.72 vs 0.75 ms)
    g.cols = std::min(count == 1 ? 4 : 8, N2);
    g.logc = 0;
    while ((1 << g.logc) < g.cols) ++g.logc;
    Scratch sc(st);
    const int64_t chunk = std::min<int64_t>(count, 65535);
    g.work[0] = sc.get<uint32_t>(size_t(chunk) << logN);
    g.work[1] = sc.get<uint32_t>(size_t(chunk) << logN);
    const size_t sm1 = size_t(N1 + 2 * padded_words(g.cols * N1)) * 4;
    const size_t sm2 = size_t(2 * N2 + 4 * padded_words(N2)) * 4;
    if (F.p < (1u << 30))
        run_ntt_launches<true>(g, F, N1, N2, count, chunk, A, lda, B, ldb, Fo, ldf, sm1, sm2, st);
    else
        run_ntt_launches<false>(g, F, N1, N2, count, chunk, A, lda, B, ldb, Fo, ldf, sm1, sm2, st);
}

template <bool LZ>
void run_ntt_launches(NttArgs g, const FieldParams& F, int N1, int N2, int64_t count,
                      int64_t chunk, const uint32_t* A, int64_t lda, const uint32_t* B,
                      int64_t ldb, uint32_t* Fo, int64_t ldf, size_t sm1, size_t sm2,
                      cudaStream_t st) {
    MMM_CUDA(cudaFuncSetAttribute(ntt_cols_fwd<LZ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sm1)));
    MMM_CUDA(cudaFuncSetAttribute(ntt_cols_inv<LZ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sm1)));
    MMM_CUDA(cudaFuncSetAttribute(ntt_rows<LZ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sm2)));
    for (int64_t c0 = 0; c0 < count; c0 += chunk) {
        const unsigned c = unsigned(std::min<int64_t>(chunk, count - c0));
        g.in[0] = A + c0 * lda;
        g.in[1] = B + c0 * ldb;
        g.ld[0] = lda;
        g.ld[1] = ldb;
        g.out = Fo + c0 * ldf;
        g.ldf = ldf;
        ntt_cols_fwd<LZ><<<dim3(N2 / g.cols, 2, c), NTT_T, sm1, st>>>(g);
        check_launch("ntt_cols_fwd");
        ntt_rows<LZ><<<dim3(N1, 1, c), NTT_T, sm2, st>>>(g, F);
        check_launch("ntt_rows");
        ntt_cols_inv<LZ><<<dim3(N2 / g.cols, 1, c), NTT_T, sm1, st>>>(g);
        check_launch("ntt_cols_inv");
    }
}

}  // namespace

template <bool LZ>
void phase_launch(NttArgs g, const FieldParams& F, int phase, int64_t start, int64_t n, size_t sm1,
                  size_t sm2, cudaStream_t st) {
    if (phase == 1) {
        MMM_CUDA(cudaFuncSetAttribute(ntt_rows<LZ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(sm2)));
        g.row0 = int(start);
        ntt_rows<LZ><<<dim3(unsigned(n), 1, 1), NTT_T, sm2, st>>>(g, F);
        check_launch("ntt_rows");
    } else {
        auto fn = phase == 0 ? ntt_cols_fwd<LZ> : ntt_cols_inv<LZ>;
        MMM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm1)));
        g.col0 = int(start);
        fn<<<dim3(unsigned(n / g.cols), phase == 0 ? 2 : 1, 1), NTT_T, sm1, st>>>(g);
        check_launch(phase == 0 ? "ntt_cols_fwd" : "ntt_cols_inv");
    }
}

// One phase of the four-step product over a slice (the sharded NTT, SURVEY
// §8f): 0 = forward columns [start, start + n) of both operands into the
// N-word workspaces, 1 = rows [start, start + n) (forward, pointwise,
// inverse), 2 = inverse columns [start, start + n) into f (natural order,
// only the positions of those columns).  Column slices are multiples of
// NTT_PHASE_COLS.
void launch_ntt_phase(const FieldParams& F, int phase, const uint32_t* a, int64_t na,
                      const uint32_t* b, int64_t nb, int64_t start, int64_t n, uint32_t* work_a,
                      uint32_t* work_b, uint32_t* f, cudaStream_t st) {
    const int64_t nf = na + nb - 1;
    const int logN = log2_len(nf);
    if (logN > 30) throw Error(ST_INVALID, "ntt: product too long");
    const NttPlan& P = get_plan(F.p, logN);
    const int N1 = 1 << P.log1, N2 = 1 << P.log2;
    NttArgs g{};
    g.P = P;
    g.in[0] = a;
    g.in[1] = b;
    g.len[0] = na;
    g.len[1] = nb;
    g.ld[0] = na;
    g.ld[1] = nb;
    g.nf = nf;
    g.work[0] = work_a;
    g.work[1] = work_b;
    g.out = f;
    g.ldf = nf;
    g.cols = std::min(NTT_PHASE_COLS, N2);
    g.logc = 0;
    while ((1 << g.logc) < g.cols) ++g.logc;
    const int64_t lim = phase == 1 ? N1 : N2;
    if (n < 0 || start < 0 || start + n > lim || (phase != 1 && (start % g.cols || n % g.cols)))
        throw Error(ST_INVALID, "ntt phase: slice outside the transform or not column-aligned");
    if (n == 0) return;
    const size_t sm1 = size_t(N1 + 2 * padded_words(g.cols * N1)) * 4;
    const size_t sm2 = size_t(2 * N2 + 4 * padded_words(N2)) * 4;
    if (F.p < (1u << 30))
        phase_launch<true>(g, F, phase, start, n, sm1, sm2, st);
    else
        phase_launch<false>(g, F, phase, start, n, sm1, sm2, st);
}

void ntt_shape(uint32_t p, int64_t nf, int64_t* n1, int64_t* n2) {
    const int logN = log2_len(nf);
    *n1 = int64_t(1) << (logN / 2);
    *n2 = int64_t(1) << (logN - logN / 2);
}

bool ntt_supported(uint32_t p, int64_t out_len) {
    if (p < 3 || (p & 1) == 0) return false;
    const int logN = log2_len(out_len);
    return logN <= 30 && ((p - 1) % (uint64_t(1) << logN)) == 0;
}

void launch_ntt_mul(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b,
                    int64_t nb, uint32_t* f, cudaStream_t st) {
    run_ntt(F, a, na, na, b, nb, nb, 1, f, na + nb - 1, st);
}

void launch_ntt_mul_batched(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                            const uint32_t* B, int64_t ldb, int64_t nb, int64_t count,
                            uint32_t* Fo, int64_t ldf, cudaStream_t st) {
    run_ntt(F, A, lda, na, B, ldb, nb, count, Fo, ldf, st);
}

}  // namespace mmm_cu
