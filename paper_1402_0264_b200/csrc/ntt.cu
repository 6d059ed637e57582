// ntt.cu -- NTT (number-theoretic FFT) multiplication over Z/pZ on sm_100a.
//
// New scope (the reference has no FFT; SPEC.md:385 lists FFT
// multiplication as a non-goal there).  Its parity anchor is uniqueness of
// the product: the result must equal oracle_mul (proj/src/oracle.cpp:8-15).
//
// Transform length N = 2^k >= na+nb-1 (needs 2^k | p-1, k <= 26), four-step
// split N = N1*N2 over the workspace w[N2*k1 + n2] (an N1 x N2 matrix):
//   K1  ntt_cols_fwd : per column n2, the N1-point forward transform of the
//                      zero-padded input x[N2*n1 + n2], times w_N^(n2*k1)
//                      (operand b's twiddle also carries N^-1 * 2^32);
//   K2  ntt_rows     : per row k1, N2-point forward transforms of both
//                      operands, the pointwise product (one Montgomery REDC,
//                      whose 2^-32 the 2^32 above cancels), a second FORWARD
//                      N2-point transform over the product, times w_N^(k1*m2);
//   K3  ntt_cols_out : per column m2, the forward N1-point transform: Z[m] at
//                      m = N2*m1 + m2, and f[n] = Z[(N - n) mod N]
//                      (the inverse transform is the forward one read
//                      backwards: NTT^-1(Y)[n] = N^-1 * NTT(Y)[-n]), so every
//                      pass uses the forward root tables.
// Each sub-transform is a Stockham autosort network whose passes run up to
// four radix-2 stages (a radix-16 unit) in registers.  The pass schedule,
// the unit -> thread map and every shared-memory offset are compile-time
// (templates over log2 length / columns / rows), so a unit's loads and
// stores are one base address plus immediates.  The first pass of a
// transform reads global memory straight into registers and the last one
// writes global memory from registers (after the four-step twiddle); in K2
// the forward transforms' last pass, the pointwise product and the product
// transform's first pass share one register unit (symmetric schedules).
// Twiddles are Shoup pairs (w, floor(w * 2^32 / p)) read through L1.
#include <map>
#include <memory>
#include <mutex>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace mmm_cu {

namespace {

constexpr int NTT_PHASE_COLS = 4;  // column granularity of the sharded phases
#ifndef NTT_KMAX
#define NTT_KMAX 4
#endif
#ifndef NTT_TMAX
#define NTT_TMAX 256
#endif
#ifndef NTT_MINB
#define NTT_MINB 2
#endif
#ifndef NTT_MINB_ROWS
#define NTT_MINB_ROWS 2
#endif
#ifndef NTT_LOGC_MAX
#define NTT_LOGC_MAX 3
#endif
#ifndef NTT_CHUNK_WORDS
#define NTT_CHUNK_WORDS (1 << 30)
#endif
#ifndef NTT_PREFER_END
#define NTT_PREFER_END 1  // 1: largest end radix (e.g. 2^10 = 4+2+4 instead of 3+4+3)
#endif
#ifndef NTT_CL_LOG
#define NTT_CL_LOG 13
#endif
constexpr int KMAX = NTT_KMAX;     // radix-2 stages per pass (radix-8 units)
constexpr int TMAX = NTT_TMAX;     // threads per CTA (end passes: one unit per thread up to TMAX)
constexpr int LOGL_MAX = 13;       // sub-transform length limit (N <= 2^26)
constexpr int LO = 10;             // four-step twiddle split: w^e = lo[e & 1023] * hi[e >> 10]

// Conditional corrections as an unsigned min: for v < 2m (m < 2^31),
// v mod m = min(v, v - m) (v - m wraps above v when v < m): one
// VIADDMNMX-class ALU op instead of a compare and a select.
__device__ __forceinline__ uint32_t umin(uint32_t a, uint32_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t shoup(uint32_t x, uint32_t w, uint32_t wp, uint32_t p) {
    const uint32_t q = __umulhi(x, wp);
    const uint32_t r = x * w - q * p;
    return umin(r, r - p);
}
// Sums and differences as min(a +- b, a +- b -+ m): IADD3 + VIADDMNMX, both on
// the ALU pipe (a plain a + b tends to become IMAD.IADD on the multiply pipe,
// the one the Shoup products saturate).
__device__ __forceinline__ uint32_t add_p(uint32_t a, uint32_t b, uint32_t p) {
    return __viaddmin_u32(a, b, a + b - p);
}
__device__ __forceinline__ uint32_t sub_p(uint32_t a, uint32_t b, uint32_t p) {
    return __viaddmin_u32(a, 0u - b, a - b + p);
}

// Butterfly halves, exact (LZ = false: canonical in and out) or lazy (LZ =
// true, p < 2^30: values in [0, 2p) in and out; Harvey's trick -- the sum
// needs one conditional subtraction of 2p, the twiddled difference none:
// a - b + 2p < 4p < 2^32 goes straight into a Shoup product, whose unreduced
// result x*w - q*p lies in [0, 2p) for any x < 2^32).
template <bool LZ>
__device__ __forceinline__ uint32_t bf_add(uint32_t a, uint32_t b, uint32_t p) {
    if (!LZ) return add_p(a, b, p);
    return __viaddmin_u32(a, b, a + b - 2 * p);
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
template <bool LZ>
__device__ __forceinline__ uint32_t bf_sub1(uint32_t a, uint32_t b, uint32_t p) {  // twiddle 1
    if (!LZ) return sub_p(a, b, p);
    return __viaddmin_u32(a, 0u - b, a - b + 2 * p);
}
__device__ __forceinline__ uint32_t canon(uint32_t v, uint32_t p) { return umin(v, v - p); }

__device__ __forceinline__ uint2 ldg2(const uint2* p) { return __ldg(p); }

// Device tables for one (p, N): the sub-transform roots and the two-level
// four-step twiddles, each value with its Shoup companion.
struct NttPlan {
    uint32_t p;
    int logN, log1, log2;  // N = N1 * N2, N1 = 2^log1 (column length), N2 = 2^log2 (row length)
    uint2* r1;     // w_N1^j,  j < N1/2
    uint2* r2;     // w_N2^j,  j < N2/2
    uint2* tlo;    // w_N^e,            e < 2^LO
    uint2* thi;    // w_N^(e << LO),    e < N >> LO
    uint2* thi_s;  // w_N^(e << LO) * N^-1 * 2^32  (operand b's forward columns)
};

// ---------------------------------------------------------- pass schedule --
// A transform of 2^logl points runs P passes of k[i] radix-2 stages each,
// k[i] <= KMAX, with k[0] == k[P-1] (so a forward transform's last register
// unit is the next transform's first: K2 keeps it in registers), as few
// passes as possible and, among those, the most balanced.
struct Sched {
    int P;
    int k[8];
    int s[8];  // first stage of each pass
};
constexpr Sched make_sched(int logl) {
    Sched r{};
    if (logl <= KMAX) {
        r.P = 1;
        r.k[0] = logl;
        return r;
    }
    for (int P = 2; P < 8; ++P) {
        int best_ke = 0, best_min = 0;
        for (int ke = KMAX; ke >= 1; --ke) {
            const int rem = logl - 2 * ke, mid = P - 2;
            const bool ok = mid == 0 ? rem == 0 : (rem >= mid && rem <= mid * KMAX);
            if (!ok) continue;
            const int mn = NTT_PREFER_END ? ke : (mid == 0 ? ke : (rem / mid < ke ? rem / mid : ke));
            if (mn > best_min) {
                best_min = mn;
                best_ke = ke;
            }
        }
        if (best_ke) {
            const int rem = logl - 2 * best_ke, mid = P - 2;
            r.P = P;
            r.k[0] = r.k[P - 1] = best_ke;
            for (int i = 0; i < mid; ++i) r.k[1 + i] = rem / mid + (i < rem % mid ? 1 : 0);
            int s = 0;
            for (int i = 0; i < P; ++i) {
                r.s[i] = s;
                s += r.k[i];
            }
            return r;
        }
    }
    return r;
}

// Shared-memory words are stored padded, one word per 32: the passes write
// groups of C*2^s consecutive words at strides 2^k * C*2^s.
__device__ __forceinline__ int PD(int i) { return i + (i >> 5); }
constexpr int padded_words(int n) { return n + (n >> 5) + 1; }

// Tile geometry: G groups (rows, in K2) x C interleaved columns x L points;
// element (g, c, n) sits at raw position g*C*L + c + C*n.  Pass I treats
// U = G*C*L/R units of R = 2^k[I] elements; unit x -> c = x mod C,
// u = (x / C) mod (L/R), g = x / (C*L/R); its element j is at raw
// g*C*L + c + C*(u + j*L/R), its output b goes to
// g*C*L + c + C*(q + 2^s*(R*pp + b)), pp = u >> s, q = u mod 2^s.
template <int LOGL_, int LOGC_, int LOGG_>
struct Geo {
    static constexpr int LOGL = LOGL_, LOGC = LOGC_, LOGG = LOGG_;
    static constexpr int L = 1 << LOGL, C = 1 << LOGC, G = 1 << LOGG;
    static constexpr int CL = C * L;
    static constexpr int WORDS = padded_words(G * CL);
    static constexpr Sched SC = make_sched(LOGL);
    static constexpr int P = SC.P;
    static constexpr int KE = SC.k[0];                    // first/last pass radix log
    static constexpr int U0 = G * C * (L >> KE);          // units of the first/last pass
    static constexpr int T = U0 < TMAX ? U0 : TMAX;       // threads per CTA
};

template <class GE, int I>
struct PassT {
    static constexpr int K = GE::SC.k[I], S = GE::SC.s[I], R = 1 << K;
    static constexpr int UR = GE::L >> K;     // units per column
    static constexpr int M = GE::C * UR;      // raw stride between a unit's elements
    static constexpr int CS = GE::C << S;     // raw stride between a unit's outputs
    static constexpr bool LIN_R = (M % 32) == 0;
    static constexpr bool LIN_W = GE::G == 1 || (GE::CL % 32) == 0;
    __device__ static __forceinline__ int c_of(int x) { return x & (GE::C - 1); }
    __device__ static __forceinline__ int u_of(int x) { return (x >> GE::LOGC) & (UR - 1); }
    __device__ static __forceinline__ int g_of(int x) { return x >> (GE::LOGC + GE::LOGL - K); }
    __device__ static __forceinline__ int rd_raw(int x) {
        return g_of(x) * GE::CL + c_of(x) + GE::C * u_of(x);
    }
    __device__ static __forceinline__ int wr_raw(int x) {
        const int u = u_of(x);
        return g_of(x) * GE::CL + c_of(x) + GE::C * (u & ((1 << S) - 1)) + R * CS * (u >> S);
    }
};

// One radix-2^K unit in registers: v[j] = element j (index pp + j*L/(R*2^S)
// at stage S) in, v[b] = output b out.  Register r at stage i holds
// (j = r >> i, low output bits bb = r & (2^i - 1)); the stage pairs r and
// r + R/2 and multiplies the difference by w_L^((pp << (S+i)) + j*(L >> (K-i))).
// The transform's last stage has twiddle 1.
template <int LOGL, int S, int K, bool LZ>
__device__ __forceinline__ void radix(uint32_t (&v)[1 << K], int pp, const uint2* __restrict__ tw,
                                      uint32_t p) {
    constexpr int R = 1 << K, L = 1 << LOGL;
    constexpr bool LASTP = S + K == LOGL;  // last pass: pp == 0, so j == 0 has twiddle 1
#pragma unroll
    for (int i = 0; i < K; ++i) {
        uint32_t w[R];
        const uint2* tb = tw + (LASTP ? 0 : (pp << (S + i)));
#pragma unroll
        for (int j = 0; j < (R >> (i + 1)); ++j) {
            const bool one = (S + i == LOGL - 1) || (LASTP && j == 0);
            uint2 t = make_uint2(1, 0);
            if (!one) t = ldg2(tb + j * (L >> (K - i)));
#pragma unroll
            for (int bb = 0; bb < (1 << i); ++bb) {
                const int r = (j << i) | bb;
                const uint32_t a0 = v[r], a1 = v[r + R / 2];
                const int o = (j << (i + 1)) | bb;
                w[o] = bf_add<LZ>(a0, a1, p);
                w[o | (1 << i)] = one ? bf_sub1<LZ>(a0, a1, p) : bf_subw<LZ>(a0, a1, t, p);
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = w[r];
    }
}

template <class PT>
__device__ __forceinline__ void lds_unit(const uint32_t* x, int xu, uint32_t (&v)[PT::R]) {
    const int raw = PT::rd_raw(xu), pd = PD(raw);
#pragma unroll
    for (int j = 0; j < PT::R; ++j)
        v[j] = PT::LIN_R ? x[pd + j * (PT::M + PT::M / 32)] : x[PD(raw + j * PT::M)];
}
template <class PT>
__device__ __forceinline__ void sts_unit(uint32_t* y, int xu, const uint32_t (&v)[PT::R]) {
    const int raw = PT::wr_raw(xu), pd = PD(raw);
#pragma unroll
    for (int b = 0; b < PT::R; ++b) {
        const int o = b * PT::CS;
        if (PT::LIN_W)
            y[pd + o + (o >> 5)] = v[b];
        else
            y[PD(raw + o)] = v[b];
    }
}

// Middle passes I in [I0, P-1): shared -> shared for NOPS operand buffers.
// In place (one buffer per operand): load + compute, barrier, store, barrier.
template <class GE, int T, int NOPS, int I, bool LZ>
__device__ __forceinline__ void mid_passes(uint32_t* const (&buf)[NOPS], const uint2* tw,
                                           uint32_t p) {
    if constexpr (I < GE::P - 1) {
        using PT = PassT<GE, I>;
        constexpr int UT = GE::G * GE::C * PT::UR;  // units per operand
        constexpr int NU = (UT + T - 1) / T;        // per thread (a middle pass may have
        constexpr bool ALL = UT % T == 0;           // a larger radix than the end passes)
        const bool act = ALL || int(threadIdx.x) < UT;
        uint32_t v[NOPS][NU][PT::R];
        if (act) {
#pragma unroll
            for (int o = 0; o < NOPS; ++o)
#pragma unroll
                for (int n = 0; n < NU; ++n) {
                    const int x = threadIdx.x + n * T;
                    lds_unit<PT>(buf[o], x, v[o][n]);
                    radix<GE::LOGL, PT::S, PT::K, LZ>(v[o][n], PT::u_of(x) >> PT::S, tw, p);
                }
        }
        __syncthreads();
        if (act) {
#pragma unroll
            for (int o = 0; o < NOPS; ++o)
#pragma unroll
                for (int n = 0; n < NU; ++n) sts_unit<PT>(buf[o], threadIdx.x + n * T, v[o][n]);
        }
        __syncthreads();
        mid_passes<GE, T, NOPS, I + 1, LZ>(buf, tw, p);
    }
}

// Programmatic dependent launch: K2 and K3 are launched with the
// programmatic-serialization attribute, so their CTAs are scheduled while the
// previous kernel's last CTAs run and wait here for its completion (and its
// memory) before touching the workspace.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Table entry by 32-bit byte offset (LOP3/SHF + a 64-bit add on the ALU pipe,
// not an IMAD.WIDE on the multiply pipe).
__device__ __forceinline__ uint2 ldg_at(const uint2* t, uint32_t byte_off) {
    return __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<uintptr_t>(t) + byte_off));
}
template <bool LZ>
__device__ __forceinline__ uint32_t twiddle(uint32_t v, uint32_t e, const uint2* lo,
                                            const uint2* hi, uint32_t p) {
    const uint2 a = ldg_at(lo, (e << 3) & (((1u << LO) - 1) << 3));
    const uint2 b = ldg_at(hi, (e >> LO) << 3);
    return shoup_l<LZ>(shoup_l<LZ>(v, a.x, a.y, p), b.x, b.y, p);
}

struct NttArgs {
    NttPlan P;
    const uint32_t* in[2];
    int64_t len[2], ld[2];
    uint32_t* work[2];  // N words per instance per operand
    uint32_t* out;
    int64_t nf, ldf;
    int col0;           // first column of this launch (sharded phases)
    int row0, row_end;  // rows [row0, row_end) of this launch
    uint32_t pinv;      // p^-1 mod 2^32 (Montgomery REDC of the pointwise product)
    bool vec_in[2];     // operand rows 16-byte aligned (vector loads in K1)
};

// K1 (OUT = false) and K3 (OUT = true): the column transforms of a tile of C
// consecutive columns.  K1: grid.y = operand; reads the zero-padded input,
// writes the twiddled workspace.  K3: reads the workspace, writes f.
template <int LOGL, int LOGC, int D, bool OUT, bool LZ>
__global__ void __launch_bounds__(Geo<LOGL, LOGC, 0>::T, NTT_MINB) ntt_cols(NttArgs g) {
    using GE = Geo<LOGL, LOGC, 0>;
    constexpr int T = GE::T;
    using P0 = PassT<GE, 0>;
    using PL = PassT<GE, GE::P - 1>;
    constexpr int NU = GE::U0 / T;
    constexpr int N2 = GE::L << D;  // row length: log2 = log1 + D
    extern __shared__ __align__(16) uint32_t sm[];
    pdl_wait();     // K3: K2's workspace (no-op when launched without PDL)
    pdl_trigger();  // let the next kernel's CTAs take the SMs this grid's tail frees
    const NttPlan& P = g.P;
    const uint32_t p = P.p;
    const int op = OUT ? 0 : blockIdx.y;
    const int64_t inst = blockIdx.z;
    const int c0 = g.col0 + blockIdx.x * GE::C;
    const uint2* tw = P.r1;
    // End passes: each thread owns V units of consecutive columns (same u),
    // so a row segment of V words moves as one vector access.
    constexpr int V = (NU % 4 == 0 && GE::C >= 4) ? 4 : ((NU % 2 == 0 && GE::C >= 2) ? 2 : 1);
    constexpr int NG = NU / V;
    using VecT = typename std::conditional<V == 4, uint4, typename std::conditional<V == 2, uint2, uint32_t>::type>::type;
    uint32_t v[NU][P0::R];
    // first pass: global -> registers
    if constexpr (!OUT) {
        const int64_t len = g.len[op];
        const bool vec_ok = g.vec_in[op];
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) {
            const int xb = V * (threadIdx.x + gi * T);
            const int c = P0::c_of(xb), u = P0::u_of(xb);
            const uint32_t* in = g.in[op] + inst * g.ld[op] + (c0 + c + u * N2);
            // element j of the group at in[j*UR*N2 + i] (immediate offsets); zero past len
            const int64_t lim64 = len - (c0 + c + int64_t(u) * N2);
            const int lim = lim64 < 0 ? 0 : (lim64 > (1 << 30) ? (1 << 30) : int(lim64));
#pragma unroll
            for (int j = 0; j < P0::R; ++j) {
                const int o = j * P0::UR * N2;
                if (V > 1 && vec_ok && o + V <= lim) {
                    const VecT t = __ldg(reinterpret_cast<const VecT*>(in + o));
#pragma unroll
                    for (int i = 0; i < V; ++i) v[gi * V + i][j] = reinterpret_cast<const uint32_t*>(&t)[i];
                } else {
#pragma unroll
                    for (int i = 0; i < V; ++i) v[gi * V + i][j] = o + i < lim ? __ldg(in + o + i) : 0u;
                }
            }
        }
    } else {
        const uint32_t* work = g.work[0] + (inst << P.logN);
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) {
            const int xb = V * (threadIdx.x + gi * T);
            const uint32_t* w = work + (c0 + P0::c_of(xb) + P0::u_of(xb) * N2);
#pragma unroll
            for (int j = 0; j < P0::R; ++j) {
                const VecT t = __ldg(reinterpret_cast<const VecT*>(w + j * P0::UR * N2));
#pragma unroll
                for (int i = 0; i < V; ++i) v[gi * V + i][j] = reinterpret_cast<const uint32_t*>(&t)[i];
            }
        }
    }
#pragma unroll
    for (int n = 0; n < NU; ++n)
        radix<LOGL, 0, P0::K, LZ>(v[n], P0::u_of(V * (threadIdx.x + (n / V) * T)), tw, p);
    if constexpr (GE::P > 1) {
#pragma unroll
        for (int n = 0; n < NU; ++n) sts_unit<P0>(sm, V * (threadIdx.x + (n / V) * T) + n % V, v[n]);
        __syncthreads();
        uint32_t* const bufs[1] = {sm};
        mid_passes<GE, T, 1, 1, LZ>(bufs, tw, p);
#pragma unroll
        for (int n = 0; n < NU; ++n) {
            lds_unit<PL>(sm, V * (threadIdx.x + (n / V) * T) + n % V, v[n]);
            radix<LOGL, PL::S, PL::K, LZ>(v[n], 0, tw, p);
        }
    }
    // last pass: registers -> global; output b of unit (c, u) is point u + b*L/R
    const int N = 1 << P.logN;
#pragma unroll
    for (int gi = 0; gi < NG; ++gi) {
        const int xb = V * (threadIdx.x + gi * T);
        const int cb = PL::c_of(xb), u = PL::u_of(xb);
        if constexpr (!OUT) {
            uint32_t* work = g.work[op] + (inst << P.logN) + (c0 + cb + u * N2);
            const uint2* hi = op == 0 ? P.thi : P.thi_s;
#pragma unroll
            for (int b = 0; b < PL::R; ++b) {  // k1 = u + b*UR, twiddle w_N^(n2*k1)
                VecT t;
#pragma unroll
                for (int i = 0; i < V; ++i) {
                    const uint32_t n2 = uint32_t(c0 + cb + i);
                    reinterpret_cast<uint32_t*>(&t)[i] =
                        twiddle<LZ>(v[gi * V + i][b], n2 * uint32_t(u + b * PL::UR), P.tlo, hi, p);
                }
                *reinterpret_cast<VecT*>(work + b * PL::UR * N2) = t;
            }
        } else {
            const int64_t nf = g.nf;
#pragma unroll
            for (int i = 0; i < V; ++i) {
                // m = N2*(u + b*UR) + c0 + c  ->  f[(N - m) mod N]; only m == 0 wraps
                const int m0 = N2 * u + c0 + cb + i;
                uint32_t* out = g.out + inst * g.ldf + (N - m0);
#pragma unroll
                for (int b = 0; b < PL::R; ++b) {
                    const int nidx = N - m0 - b * PL::UR * N2;
                    if (m0 == 0 && b == 0)
                        g.out[inst * g.ldf] = canon(v[gi * V + i][b], p);
                    else if (nidx < nf)
                        out[-b * PL::UR * N2] = canon(v[gi * V + i][b], p);
                }
            }
        }
    }
}

// K2: per row k1 (G rows per CTA): forward transforms of both operands,
// pointwise product, forward transform of the product, twiddle w_N^(k1*m2).
template <int LOGL, int LOGG, bool LZ>
__global__ void __launch_bounds__(Geo<LOGL, 0, LOGG>::U0, NTT_MINB_ROWS) ntt_rows(NttArgs g) {
    using GE = Geo<LOGL, 0, LOGG>;
    constexpr int T = GE::U0;
    static_assert(T <= 1024, "one end-pass unit per operand per thread");
    using P0 = PassT<GE, 0>;
    using PL = PassT<GE, GE::P - 1>;
    static_assert(P0::K == PL::K, "symmetric schedule");
    extern __shared__ __align__(16) uint32_t sm[];
    pdl_wait();  // K1's workspace
    pdl_trigger();
    const NttPlan& P = g.P;
    const uint32_t p = P.p;
    constexpr int N2 = GE::L;
    const int64_t inst = blockIdx.z;
    const int x = threadIdx.x;
    const int u = P0::u_of(x);
    const int k1 = g.row0 + blockIdx.x * GE::G + P0::g_of(x);
    const bool valid = k1 < g.row_end;
    uint32_t* wa = g.work[0] + (inst << P.logN) + (k1 * N2 + u);
    const uint32_t* wb = g.work[1] + (inst << P.logN) + (k1 * N2 + u);
    const uint2* tw = P.r2;
    uint32_t va[P0::R], vb[P0::R];
#pragma unroll
    for (int j = 0; j < P0::R; ++j) {
        va[j] = valid ? wa[j * P0::UR] : 0u;
        vb[j] = valid ? __ldg(wb + j * P0::UR) : 0u;
    }
    radix<LOGL, 0, P0::K, LZ>(va, u, tw, p);
    radix<LOGL, 0, P0::K, LZ>(vb, u, tw, p);
    uint32_t* const bufs[2] = {sm, sm + GE::WORDS};
    if constexpr (GE::P > 1) {
        sts_unit<P0>(bufs[0], x, va);
        sts_unit<P0>(bufs[1], x, vb);
        __syncthreads();
        mid_passes<GE, T, 2, 1, LZ>(bufs, tw, p);
        lds_unit<PL>(bufs[0], x, va);
        lds_unit<PL>(bufs[1], x, vb);
        radix<LOGL, PL::S, PL::K, LZ>(va, 0, tw, p);
        radix<LOGL, PL::S, PL::K, LZ>(vb, 0, tw, p);
    }
    // pointwise: redc(a*b) = a*b*2^-32 (a, b < 2p: a*b < 4p^2 < p*2^32)
#pragma unroll
    for (int j = 0; j < P0::R; ++j) {
        const uint64_t t = uint64_t(va[j]) * vb[j];
        const uint32_t m = uint32_t(t) * g.pinv;
        const uint32_t r = uint32_t(t >> 32) - __umulhi(m, p);
        va[j] = umin(r, r + p);
    }
    // the product transform (forward); its first unit is this thread's unit
    radix<LOGL, 0, P0::K, LZ>(va, u, tw, p);
    if constexpr (GE::P > 1) {
        __syncthreads();  // every thread has read bufs[0] in the last pass
        sts_unit<P0>(bufs[0], x, va);
        __syncthreads();
        uint32_t* const one[1] = {bufs[0]};
        mid_passes<GE, T, 1, 1, LZ>(one, tw, p);
        lds_unit<PL>(bufs[0], x, va);
        radix<LOGL, PL::S, PL::K, LZ>(va, 0, tw, p);
    }
    if (valid) {
        const uint32_t e0 = uint32_t(k1) * uint32_t(u), de = uint32_t(k1) * PL::UR;
#pragma unroll
        for (int b = 0; b < PL::R; ++b)  // m2 = u + b*UR, twiddle w_N^(k1*m2)
            wa[b * PL::UR] = twiddle<LZ>(va[b], e0 + b * de, P.tlo, P.thi, p);
    }
}

// ------------------------------------------------- per-length launch table --
// Columns per CTA in the column passes: C*L <= 8192 words (32 KB), C <= 8.
constexpr int main_logc(int logl) {
    const int c = NTT_CL_LOG - logl;
    const int m = logl < NTT_LOGC_MAX ? logl : NTT_LOGC_MAX;
    return c < 0 ? 0 : (c > m ? m : c);
}
// Rows per CTA in K2: at least 128 threads (one radix unit per operand each).
constexpr int rows_logg(int logl) {
    const int ke = make_sched(logl).k[0];
    const int g = 7 - (logl - ke);
    return g < 0 ? 0 : g;
}

using ColsFn = void (*)(NttArgs);
struct ColsKernel {
    ColsFn fn;
    int threads, cols;
    size_t smem;
};

template <int LOGL, int LOGC, int D, bool OUT, bool LZ>
ColsKernel cols_kernel() {
    using GE = Geo<LOGL, LOGC, 0>;
    const size_t smem = GE::P > 1 ? size_t(GE::WORDS) * 4 : 0;
    ColsKernel k{ntt_cols<LOGL, LOGC, D, OUT, LZ>, GE::T, GE::C, smem};
    if (smem > 48 * 1024)
        MMM_CUDA(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    return k;
}

template <int LOGL, bool OUT, bool LZ>
ColsKernel cols_for(bool phase, int d) {
    constexpr int LM = main_logc(LOGL);
    constexpr int LP = LOGL < 2 ? LOGL : 2;  // phases: NTT_PHASE_COLS columns (N2 >= L)
    if (phase) return d ? cols_kernel<LOGL, LP, 1, OUT, LZ>() : cols_kernel<LOGL, LP, 0, OUT, LZ>();
    return d ? cols_kernel<LOGL, LM, 1, OUT, LZ>() : cols_kernel<LOGL, LM, 0, OUT, LZ>();
}

struct RowsKernel {
    ColsFn fn;
    int threads, rows;
    size_t smem;
};
template <int LOGL, bool LZ>
RowsKernel rows_for() {
    using GE = Geo<LOGL, 0, rows_logg(LOGL)>;
    const size_t smem = GE::P > 1 ? size_t(2 * GE::WORDS) * 4 : 0;
    RowsKernel k{ntt_rows<LOGL, rows_logg(LOGL), LZ>, GE::U0, GE::G, smem};
    if (smem > 48 * 1024)
        MMM_CUDA(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    return k;
}

template <bool OUT, bool LZ>
ColsKernel pick_cols(int logl, int log2, bool phase) {
    switch (logl) {
#define MMM_NTT_CASE(n) \
    case n:             \
        return cols_for<n, OUT, LZ>(phase, log2 - logl);
        MMM_NTT_CASE(1) MMM_NTT_CASE(2) MMM_NTT_CASE(3) MMM_NTT_CASE(4) MMM_NTT_CASE(5)
        MMM_NTT_CASE(6) MMM_NTT_CASE(7) MMM_NTT_CASE(8) MMM_NTT_CASE(9) MMM_NTT_CASE(10)
        MMM_NTT_CASE(11) MMM_NTT_CASE(12) MMM_NTT_CASE(13)
#undef MMM_NTT_CASE
    }
    throw Error(ST_INVALID, "ntt: transform too long");
}
template <bool LZ>
RowsKernel pick_rows(int logl) {
    switch (logl) {
#define MMM_NTT_CASE(n) \
    case n:             \
        return rows_for<n, LZ>();
        MMM_NTT_CASE(1) MMM_NTT_CASE(2) MMM_NTT_CASE(3) MMM_NTT_CASE(4) MMM_NTT_CASE(5)
        MMM_NTT_CASE(6) MMM_NTT_CASE(7) MMM_NTT_CASE(8) MMM_NTT_CASE(9) MMM_NTT_CASE(10)
        MMM_NTT_CASE(11) MMM_NTT_CASE(12) MMM_NTT_CASE(13)
#undef MMM_NTT_CASE
    }
    throw Error(ST_INVALID, "ntt: transform too long");
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

std::vector<uint2> powers(uint32_t w, size_t n, uint32_t p, uint32_t scale = 1) {
    std::vector<uint2> v(n);
    uint64_t x = scale % p;
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
    const uint32_t w1 = pow_mod(wN, uint64_t(1) << P.log2, p);  // order N1
    const uint32_t w2 = pow_mod(wN, uint64_t(1) << P.log1, p);  // order N2
    const uint32_t ninv = pow_mod(uint32_t(N % p), p - 2, p);
    const uint32_t r32 = uint32_t((uint64_t(1) << 32) % p);
    const uint32_t bscale = uint32_t(uint64_t(ninv) * r32 % p);  // N^-1 * 2^32
    auto upload = [](const std::vector<uint2>& v) {
        uint2* d = nullptr;
        MMM_CUDA(cudaMalloc(&d, std::max<size_t>(v.size(), 1) * sizeof(uint2)));
        MMM_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(uint2), cudaMemcpyHostToDevice));
        return d;
    };
    const size_t n1h = std::max<size_t>((size_t(1) << P.log1) / 2, 1);
    const size_t n2h = std::max<size_t>((size_t(1) << P.log2) / 2, 1);
    P.r1 = upload(powers(w1, n1h, p));
    P.r2 = upload(powers(w2, n2h, p));
    const size_t nlo = size_t(1) << LO, nhi = std::max<size_t>(N >> LO, 1);
    P.tlo = upload(powers(wN, nlo, p));
    P.thi = upload(powers(pow_mod(wN, nlo, p), nhi, p));
    P.thi_s = upload(powers(pow_mod(wN, nlo, p), nhi, p, bscale));
    const NttPlan& ref = *plan;
    g_plans.plans.emplace(key, std::move(plan));
    return ref;
}

}  // namespace

void release_plans() {
    std::lock_guard<std::mutex> lk(g_plans.mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& kv : g_plans.plans) {
        cudaSetDevice(std::get<0>(kv.first));
        for (uint2* t : {kv.second->r1, kv.second->r2, kv.second->tlo, kv.second->thi,
                         kv.second->thi_s})
            cudaFree(t);
    }
    g_plans.plans.clear();
    cudaSetDevice(cur);
}

namespace {

int log2_len(int64_t nf) {
    int k = 2;
    while ((int64_t(1) << k) < nf) ++k;
    return k;
}

uint32_t p_inverse(uint32_t p) {  // p^-1 mod 2^32, odd p
    uint32_t inv = p;
    for (int i = 0; i < 5; ++i) inv *= 2u - p * inv;
    return inv;
}

void launch_pdl(ColsFn fn, dim3 grid, int threads, size_t smem, cudaStream_t st, NttArgs g) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(unsigned(threads));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MMM_CUDA(cudaLaunchKernelEx(&cfg, fn, g));
}

template <bool LZ>
void run_ntt_launches(NttArgs g, int64_t count, int64_t chunk, const uint32_t* A, int64_t lda,
                      const uint32_t* B, int64_t ldb, uint32_t* Fo, int64_t ldf, cudaStream_t st) {
    const int N1 = 1 << g.P.log1, N2 = 1 << g.P.log2;
    const ColsKernel kf = pick_cols<false, LZ>(g.P.log1, g.P.log2, false);
    const ColsKernel ko = pick_cols<true, LZ>(g.P.log1, g.P.log2, false);
    const RowsKernel kr = pick_rows<LZ>(g.P.log2);
    g.col0 = 0;
    g.row0 = 0;
    g.row_end = N1;
    for (int64_t c0 = 0; c0 < count; c0 += chunk) {
        const unsigned c = unsigned(std::min<int64_t>(chunk, count - c0));
        g.in[0] = A + c0 * lda;
        g.in[1] = B + c0 * ldb;
        g.vec_in[0] = (reinterpret_cast<uintptr_t>(g.in[0]) % 16 == 0) && (lda % 4 == 0 || c == 1);
        g.vec_in[1] = (reinterpret_cast<uintptr_t>(g.in[1]) % 16 == 0) && (ldb % 4 == 0 || c == 1);
        g.ld[0] = lda;
        g.ld[1] = ldb;
        g.out = Fo + c0 * ldf;
        g.ldf = ldf;
        kf.fn<<<dim3(N2 / kf.cols, 2, c), kf.threads, kf.smem, st>>>(g);
        check_launch("ntt_cols_fwd", dim3(N2 / kf.cols, 2, c), dim3(kf.threads));
        launch_pdl(kr.fn, dim3((N1 + kr.rows - 1) / kr.rows, 1, c), kr.threads, kr.smem, st, g);
        check_launch("ntt_rows", dim3((N1 + kr.rows - 1) / kr.rows, 1, c), dim3(kr.threads));
        launch_pdl(ko.fn, dim3(N2 / ko.cols, 1, c), ko.threads, ko.smem, st, g);
        check_launch("ntt_cols_out", dim3(N2 / ko.cols, 1, c), dim3(ko.threads));
    }
}

NttArgs base_args(const NttPlan& P, int64_t nf) {
    NttArgs g{};
    g.P = P;
    g.nf = nf;
    g.pinv = p_inverse(P.p);
    return g;
}

void run_ntt(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na, const uint32_t* B,
             int64_t ldb, int64_t nb, int64_t count, uint32_t* Fo, int64_t ldf, cudaStream_t st) {
    const int64_t nf = na + nb - 1;
    const int logN = log2_len(nf);
    if (logN > 2 * LOGL_MAX) throw Error(ST_INVALID, "ntt: product too long");
    const NttPlan& P = get_plan(F.p, logN);
    NttArgs g = base_args(P, nf);
    g.len[0] = na;
    g.len[1] = nb;
    Scratch sc(st);
    // instances per launch group: the two N-word workspaces of a group stay
    // L2-resident (2 x 16 MB at the default), so the row pass reads what the
    // column pass wrote from L2 instead of HBM
    int64_t chunk_words = int64_t(NTT_CHUNK_WORDS);
    if (const char* e = getenv("MMM_NTT_CHUNK_WORDS")) chunk_words = atoll(e);  // tools/ntt_sweep
    const int64_t chunk =
        std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(count, 65535), chunk_words >> logN));
    g.work[0] = sc.get<uint32_t>(size_t(chunk) << logN);
    g.work[1] = sc.get<uint32_t>(size_t(chunk) << logN);
    if (F.p < (1u << 30))
        run_ntt_launches<true>(g, count, chunk, A, lda, B, ldb, Fo, ldf, st);
    else
        run_ntt_launches<false>(g, count, chunk, A, lda, B, ldb, Fo, ldf, st);
}

template <bool LZ>
void phase_launch(NttArgs g, int phase, int64_t start, int64_t n, cudaStream_t st) {
    if (phase == 1) {
        const RowsKernel kr = pick_rows<LZ>(g.P.log2);
        g.row0 = int(start);
        g.row_end = int(start + n);
        kr.fn<<<dim3(unsigned((n + kr.rows - 1) / kr.rows), 1, 1), kr.threads, kr.smem, st>>>(g);
        check_launch("ntt_rows", dim3(unsigned((n + kr.rows - 1) / kr.rows)), dim3(kr.threads));
    } else {
        const ColsKernel k = phase == 0 ? pick_cols<false, LZ>(g.P.log1, g.P.log2, true)
                                        : pick_cols<true, LZ>(g.P.log1, g.P.log2, true);
        g.col0 = int(start);
        k.fn<<<dim3(unsigned(n / k.cols), phase == 0 ? 2 : 1, 1), k.threads, k.smem, st>>>(g);
        check_launch(phase == 0 ? "ntt_cols_fwd" : "ntt_cols_out",
                     dim3(unsigned(n / k.cols), phase == 0 ? 2 : 1, 1), dim3(k.threads));
    }
}

}  // namespace

// One phase of the four-step product over a slice (the sharded NTT, SURVEY
// §8f): 0 = forward columns [start, start + n) of both operands into the
// N-word workspaces, 1 = rows [start, start + n) (forward, pointwise,
// forward of the product), 2 = output columns [start, start + n) into f:
// the positions n with (N - n) mod N2 in the slice (each f position is
// written by exactly one column).  Column slices are multiples of
// NTT_PHASE_COLS.
void launch_ntt_phase(const FieldParams& F, int phase, const uint32_t* a, int64_t na,
                      const uint32_t* b, int64_t nb, int64_t start, int64_t n, uint32_t* work_a,
                      uint32_t* work_b, uint32_t* f, cudaStream_t st) {
    const int64_t nf = na + nb - 1;
    const int logN = log2_len(nf);
    if (logN > 2 * LOGL_MAX) throw Error(ST_INVALID, "ntt: product too long");
    const NttPlan& P = get_plan(F.p, logN);
    const int N1 = 1 << P.log1, N2 = 1 << P.log2;
    NttArgs g = base_args(P, nf);
    g.in[0] = a;
    g.in[1] = b;
    g.vec_in[0] = reinterpret_cast<uintptr_t>(a) % 16 == 0;
    g.vec_in[1] = reinterpret_cast<uintptr_t>(b) % 16 == 0;
    g.len[0] = na;
    g.len[1] = nb;
    g.ld[0] = na;
    g.ld[1] = nb;
    g.work[0] = work_a;
    g.work[1] = work_b;
    g.out = f;
    g.ldf = nf;
    const int cols = std::min(NTT_PHASE_COLS, N2);
    const int64_t lim = phase == 1 ? N1 : N2;
    if (n < 0 || start < 0 || start + n > lim || (phase != 1 && (start % cols || n % cols)))
        throw Error(ST_INVALID, "ntt phase: slice outside the transform or not column-aligned");
    if (n == 0) return;
    if (F.p < (1u << 30))
        phase_launch<true>(g, phase, start, n, st);
    else
        phase_launch<false>(g, phase, start, n, st);
}

void ntt_shape(uint32_t p, int64_t nf, int64_t* n1, int64_t* n2) {
    const int logN = log2_len(nf);
    *n1 = int64_t(1) << (logN / 2);
    *n2 = int64_t(1) << (logN - logN / 2);
}

bool ntt_supported(uint32_t p, int64_t out_len) {
    if (p < 3 || (p & 1) == 0) return false;
    const int logN = log2_len(out_len);
    return logN <= 2 * LOGL_MAX && ((p - 1) % (uint64_t(1) << logN)) == 0;
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
