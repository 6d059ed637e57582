// gcd.cu -- Euclidean GCD over Z/pZ on sm_100a.
//
// Result: exactly oracle_gcd (proj/src/oracle.cpp:69-78), the monic gcd.
// Structure: the paper's blocked GCD (Alg. 9-10), simulated by
// run_gcd's optimized variant (proj/src/gcd.cpp:116-330): a run of head
// eliminations is folded into a 2x2 matrix of offset polynomials
// (UpdateMatrix, gcd.cpp:124-157) which every block then applies to its part
// of both operands.  B200-first re-design:
//
//  * Fraction-free steps.  U <- y*U - x*X^k*V (x, y the leads) evaluated as
//    one Montgomery reduction of y*u + (p-x)*v: no field inverse per step;
//    the operands stay associates of the oracle's remainders, so the final
//    monic gcd is bit-identical.  For p < 2^29 the reduction is lazy
//    (values in [0, 2p), no correction), which keeps a step at 5 integer ops.
//  * Top-aligned windows in registers.  With u[t] = U[deg U - t] the update
//    is u[t] <- y*u[t] - x*v[t]: lane-aligned, no shuffles; only the
//    renormalisation after a degree drop (u[t] <- u[t+z]) moves data.  Warp 0
//    of CTA 0 runs the whole step chain on 128-word windows of both operands
//    held 4 words per lane, and logs each step (x, y, z, which operand).
//  * The matrix in the same top-aligned form.  Pu[t] satisfies
//    u[t] = sum_e Pu1[e] a0[t+e] + sum_e Pu2[e] b0[t+e]; it obeys the same
//    recurrence as the window (Pu <- y*Pu - x*Pv) and shifts right by z when
//    the window shifts left.  Warps 1 and 2 replay the step log, one matrix
//    column each, concurrently with the chain.
//  * Grid-wide apply.  The matrix is published to global memory and every
//    CTA applies it to its slice of both operands with the register-tiled
//    convolution of conv.cuh (L2-resident ping-pong buffers); one grid
//    barrier before and one after.  The role rule is the oracle's: the
//    dividend is reduced while deg(dividend) >= deg(divisor)
//    (oracle.cpp:58-66), then roles swap (oracle.cpp:74-75); a zero dividend
//    ends the run with the divisor as gcd, a degree-0 divisor with gcd 1
//    (gcd.cpp:191-199).
#include <cooperative_groups.h>

#include "common.cuh"
#include "conv.cuh"

#include <cstdio>
#include <map>
#include <mutex>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace mmm_cu {

constexpr int GCD_T = 256;         // threads per CTA
#ifndef GCD_GE
#define GCD_GE 2
#endif
#ifndef GCD_PE
#define GCD_PE 2
#endif
constexpr int GE = GCD_GE;         // window words per lane
constexpr int W1 = 32 * GE;        // window words per operand
constexpr int PE = GCD_PE;         // matrix words per lane per polynomial
constexpr int PL = 32 * PE;        // matrix capacity (support < PL)
constexpr int LOGCAP = 512;        // log entries per batch (<= PL + 1 in practice)
constexpr int BIG = 1 << 30;
#ifndef GCD_REPLAY_SIMPLE
#define GCD_REPLAY_SIMPLE 0  // 0: pair loop + prefetch; 2: one poll loop per pair (5 % slower in the kernel); 1: one entry per iteration (1.8x slower replay)
#endif
#ifndef GCD_CHAIN_LA
#define GCD_CHAIN_LA 0  // steady state: 1 = scalar-lookahead rounds (faster alone, slower in the kernel)
#endif       // "validity unbounded": window covers the operand

struct StepLog {
    uint32_t x, y;
    int z;       // renormalisation shift of the reduced operand
    int u_is_a;  // 1: A was reduced by B, 0: B by A
};

// Published per batch by CTA 0 into a ring slot, read by the bulk CTAs.
// All 32-bit fields, in the order of the record's meta words, so that lane l
// of the bulk's polling warp stores word l with one shared store (a switch
// over the fields diverges and costs ~1 us of serial address conversions).
struct BatchMeta {
    int da0, db0;        // exact degrees at batch start (-1: zero operand)
    int da1, db1;        // degree bounds after the batch (-1: vanished)
    int steps, term, dividend_a, err;
    int sa, sb;          // total shifts of A and B (top moves)
    int hi[4];           // highest nonzero index of Pa1, Pa2, Pb1, Pb2
    int tpub_lo, tpub_hi;  // MMM_GCD_STATS: %globaltimer at publication
    int minprog;         // min bulk progress the head saw (bulk ring guard)
};

constexpr int RING = 4;  // published batch records in flight
constexpr int NBUF = 4;  // state buffers: batch j reads j % NBUF, writes (j+1) % NBUF
constexpr int META_W = 17;             // meta words of a batch record
constexpr int REC_W = 4 * PL + META_W;  // record: Pa1, Pa2, Pb1, Pb2 (canonical), meta

// Cross-CTA data are tagged words, (tag << 32) | value, written and read with
// single-copy-atomic 64-bit relaxed accesses: a reader polls the very words it
// needs until their tag is the one it expects, so no flag, fence or counter
// sits between a producer's store and a consumer's use (one L2 round trip).
// State S_j (the operands after j batches) carries tag j + 1; batch j's record
// tag j + 1.
struct GcdArgs {
    const uint32_t* a;
    const uint32_t* b;
    long long na, nb;
    uint64_t* XA[NBUF];   // tagged state of A
    uint64_t* XB[NBUF];
    uint64_t* rec;        // RING tagged batch records (REC_W words each)
    long long cap;        // words per state buffer
    unsigned* prog;       // per bulk CTA: batches finished (ring-reuse guards only; a
                          // shared counter would serialise 147 atomics per batch)
    uint32_t* g;
    int64_t* ng;
    int M;                // steps per batch (the program parameter s)
    FieldParams F;
    long long* stats;     // optional (MMM_GCD_STATS)
    int dbg;              // MMM_GCD_DEBUG bits (timing experiments)
};

namespace {

// Field flavour of the chain, fixed at compile time so the hot loops carry
// no fallback branch: MODE 0 = odd p < 2^29, lazy residues in [0, 2p);
// MODE 1 = odd p, canonical; MODE 2 = p = 2.
struct Fld {
    uint32_t p, pinv;
};

template <int MODE>
struct Arith {
    // y*a - x*b (negx = -x) times 2^-32 (odd p); canonical unless MODE 0.
    static __device__ __forceinline__ uint32_t comb(uint32_t y, uint32_t a, uint32_t negx,
                                                     uint32_t b, Fld f) {
        const uint64_t t = uint64_t(y) * a + uint64_t(negx) * b;
        if (MODE == 2) return uint32_t(t & 1u);
        const uint32_t m = uint32_t(t) * f.pinv;
        const uint32_t hi = uint32_t(t >> 32), mp = __umulhi(m, f.p);
        if (MODE == 0) return hi - mp + f.p;  // t < 8p^2 < p*2^32 for p < 2^29: in (0, 2p)
        const uint32_t r = hi - mp;
        return hi < mp ? r + f.p : r;
    }
    // (a*x + b*y + c*z) * 2^-32, MODE 0 only: a, b, c canonical, x, y, z lazy
    // (< 2p), so t < 6p^2 < p*2^32 and the lazy result lies in (0, 2p).
    static __device__ __forceinline__ uint32_t comb3(uint32_t a, uint32_t x, uint32_t b, uint32_t y,
                                                      uint32_t c, uint32_t z, Fld f) {
        const uint64_t t = uint64_t(a) * x + uint64_t(b) * y + uint64_t(c) * z;
        const uint32_t m = uint32_t(t) * f.pinv;
        return uint32_t(t >> 32) - __umulhi(m, f.p) + f.p;
    }
    // a*b * 2^-32, canonical (MODE 0 operands < 2p)
    static __device__ __forceinline__ uint32_t mont(uint32_t a, uint32_t b, Fld f) {
        const uint64_t t = uint64_t(a) * b;
        const uint32_t m = uint32_t(t) * f.pinv;
        const uint32_t r = uint32_t(t >> 32) - __umulhi(m, f.p) + f.p;
        return r >= f.p ? r - f.p : r;
    }
    static __device__ __forceinline__ bool nz(uint32_t v, uint32_t p) {
        return MODE == 0 ? (v != 0u && v != p) : v != 0u;
    }
    static __device__ __forceinline__ uint32_t neg(uint32_t x, uint32_t p) {
        return MODE == 0 ? 2u * p - x : (x ? p - x : 0u);
    }
    static __device__ __forceinline__ uint32_t canon(uint32_t v, uint32_t p) {
        return MODE == 0 ? (v >= p ? v - p : v) : v;
    }
};

// Release/acquire on a shared-memory flag (no full sequentially-consistent
// fence per step: MEMBAR.SC would stall the chain warp every elimination).
__device__ __forceinline__ void st_release_cta(volatile int* p, int v) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(const_cast<int*>(p)));
    asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cta(volatile int* p) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(const_cast<int*>(p)));
    int v;
    asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint64_t ld_rlx64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_tag(uint64_t* p, uint32_t v, unsigned tag) {
#if GCD_WEAK_TAG_STORES
    __stcg(reinterpret_cast<unsigned long long*>(p), (uint64_t(tag) << 32) | v);
#else
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"((uint64_t(tag) << 32) | v)
                 : "memory");
#endif
}
// The value of a tagged word already loaded as w, re-polled until it carries `tag`.
__device__ __forceinline__ uint32_t tag_resolve(const uint64_t* p, uint64_t w, unsigned tag) {
    while (unsigned(w >> 32) != tag) {
#ifdef GCD_POLL_SLEEP
        __nanosleep(GCD_POLL_SLEEP);
#endif
        w = ld_rlx64(p);
    }
    return uint32_t(w);
}
// K tagged words already loaded into w[]: re-poll every stale one together
// (one round trip per round, not one per word) until all carry `tag`.
template <int K>
__device__ __forceinline__ void tag_resolve_all(const uint64_t* const (&p)[K], uint64_t (&w)[K],
                                                unsigned tag) {
    for (;;) {
        bool ok = true;
#pragma unroll
        for (int k = 0; k < K; ++k) ok &= unsigned(w[k] >> 32) == tag;
        if (ok) return;
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (unsigned(w[k] >> 32) != tag) w[k] = ld_rlx64(p[k]);
    }
}
__device__ __forceinline__ uint32_t ld_tag(const uint64_t* p, unsigned tag) {
    return tag_resolve(p, ld_rlx64(p), tag);
}
__device__ __forceinline__ uint32_t bcast(uint32_t v) { return __shfl_sync(0xffffffffu, v, 0); }
__device__ __forceinline__ uint32_t from_lane(uint32_t v, int l) {
    return __shfl_sync(0xffffffffu, v, l);
}

// w[t] <- w[t + z] (top-aligned left shift), t = slot*32 + lane; z uniform.
template <int N>
__device__ __forceinline__ void shift_left(uint32_t (&w)[N], int z) {
    const int lane = threadIdx.x & 31;
    for (; z >= 32; z -= 32) {
#pragma unroll
        for (int e = 0; e < N - 1; ++e) w[e] = w[e + 1];
        w[N - 1] = 0u;
    }
    const int src = (lane + z) & 31;
    const bool carry = lane + z >= 32;
    uint32_t r[N];
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = __shfl_sync(0xffffffffu, w[e], src);
#pragma unroll
    for (int e = 0; e < N; ++e) w[e] = carry ? (e + 1 < N ? r[e + 1] : 0u) : r[e];
}

// w[t] <- w[t - z] (right shift, zeros enter at t < z); z uniform.
template <int N>
__device__ __forceinline__ void shift_right(uint32_t (&w)[N], int z) {
    const int lane = threadIdx.x & 31;
    for (; z >= 32; z -= 32) {
#pragma unroll
        for (int e = N - 1; e > 0; --e) w[e] = w[e - 1];
        w[0] = 0u;
    }
    const int src = (lane - z) & 31;
    const bool borrow = lane < z;
    uint32_t r[N];
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = __shfl_sync(0xffffffffu, w[e], src);
#pragma unroll
    for (int e = N - 1; e >= 0; --e) w[e] = borrow ? (e > 0 ? r[e - 1] : 0u) : r[e];
}

// Fast one-word shifts (the common renormalisation), touching only the first
// `na` slots (warp-uniform): words beyond them are dead (past the validity
// of a window, or past the support of a matrix row).
template <int N>
__device__ __forceinline__ void shift_left1(uint32_t (&w)[N], int na) {
    const int lane = threadIdx.x & 31;
    uint32_t r[N];
#pragma unroll
    for (int e = 0; e < N; ++e)
        if (e < na) r[e] = __shfl_sync(0xffffffffu, w[e], (lane + 1) & 31);
#pragma unroll
    for (int e = 0; e < N; ++e)
        if (e < na) w[e] = lane == 31 ? (e + 1 < N && e + 1 < na ? r[e + 1] : 0u) : r[e];
}
template <int N>
__device__ __forceinline__ void shift_right1(uint32_t (&w)[N], int na) {
    const int lane = threadIdx.x & 31;
    uint32_t r[N];
#pragma unroll
    for (int e = 0; e < N; ++e)
        if (e < na) r[e] = __shfl_sync(0xffffffffu, w[e], (lane - 1) & 31);
#pragma unroll
    for (int e = N - 1; e >= 0; --e)
        if (e < na) w[e] = lane == 0 ? (e > 0 ? r[e - 1] : 0u) : r[e];
}

// o[t] = w[t + K] (top-aligned copy shifted left by a constant; zeros enter).
template <int K, int N>
__device__ __forceinline__ void shl_copy(const uint32_t (&w)[N], uint32_t (&o)[N]) {
    const int lane = threadIdx.x & 31;
    uint32_t r[N];
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = __shfl_sync(0xffffffffu, w[e], (lane + K) & 31);
#pragma unroll
    for (int e = 0; e < N; ++e) o[e] = lane + K >= 32 ? (e + 1 < N ? r[e + 1] : 0u) : r[e];
}
// o[t] = w[t - K] (right-shifted copy; zeros enter at t < K).
template <int K, int N>
__device__ __forceinline__ void shr_copy(const uint32_t (&w)[N], uint32_t (&o)[N]) {
    const int lane = threadIdx.x & 31;
    uint32_t r[N];
#pragma unroll
    for (int e = 0; e < N; ++e) r[e] = __shfl_sync(0xffffffffu, w[e], (lane - K) & 31);
#pragma unroll
    for (int e = 0; e < N; ++e) o[e] = lane < K ? (e > 0 ? r[e - 1] : 0u) : r[e];
}

// First t >= from with w[t] != 0 (warp-uniform), or -1.
template <int MODE, int N>
__device__ __forceinline__ int first_nz(const uint32_t (&w)[N], int from, uint32_t p) {
    const int lane = threadIdx.x & 31;
    int z = -1;
#pragma unroll
    for (int e = 0; e < N; ++e) {
        const unsigned m = __ballot_sync(0xffffffffu, Arith<MODE>::nz(w[e], p) && e * 32 + lane >= from);
        if (z < 0 && m) z = e * 32 + __ffs(m) - 1;
    }
    return z;
}

// Log entry, stored by every lane of the chain warp (same address, same
// value: no divergence, no fence).  Single step: (x, y, 0, meta), the
// dividend u <- y*u - x*v shifted by z.  Fused pair (MODE 0): (alpha, beta,
// gamma, meta), u <- alpha*u[t+2] + beta*v[t+2] + gamma*v[t+1] shifted by a
// further z - 2.  meta = tag << 10 | fused << 9 | u_is_a << 8 | z (z < 256):
// the 22-bit batch tag publishes the entry to the replay warps, which poll it,
// and retires older batches' entries without clearing the log (cleared only
// when the tag wraps).
constexpr unsigned LOG_FUSED = 1u << 9, LOG_UA = 1u << 8, LOG_Z = 0xFFu;
constexpr unsigned TAG_MASK = (1u << 22) - 1;
__device__ __forceinline__ unsigned batch_tag(int j) { return unsigned(j) % TAG_MASK + 1u; }
// The log is addressed through its 32-bit shared-window base (taken once:
// converting a generic pointer reads SR_CgaCtaId, a slow S2R, every time).
__device__ __forceinline__ unsigned log_base(const StepLog* log) {
    return static_cast<unsigned>(__cvta_generic_to_shared(const_cast<StepLog*>(log)));
}
__device__ __forceinline__ unsigned log_seq(int /*i*/, unsigned tag) { return tag; }
#ifdef GCD_TRACE  // tools/chain_bench2: per-entry write / replay clocks
__device__ long long g_tw[LOGCAP], g_tr[LOGCAP], g_tp[LOGCAP], g_ta[LOGCAP], g_tb[LOGCAP];
#endif
__device__ __forceinline__ void log_entry(unsigned lb, int i, unsigned par, uint32_t c0, uint32_t c1,
                                          uint32_t c2, unsigned meta) {
#ifdef GCD_TRACE
    if ((threadIdx.x & 31) == 0) g_tw[i] = clock64();
#endif
    const unsigned a = lb + unsigned(i) * 16u;
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(c0), "r"(c1), "r"(c2),
                 "r"(meta | (log_seq(i, par) << 10)));
}
__device__ __forceinline__ uint4 log_get(unsigned lb, int i) {
    const unsigned a = lb + unsigned(i) * 16u;
    uint4 v;
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a)
                 : "memory");
    return v;
}

// Renormalisation after a comb whose candidate lead u[0] vanished: the first
// nonzero t >= 1 within the valid words `vmin` and the matrix room `room`.
// Returns the shift (du lowered by it; du = -1 if the whole operand vanished).
template <int MODE>
__device__ __forceinline__ int renorm(uint32_t (&u)[GE], int& du, int vmin, int room, bool& stop,
                                      uint32_t p) {
    int z = first_nz<MODE>(u, 1, p);
    if (z < 0 || z >= vmin) {
        if (vmin >= BIG) {  // the window held the whole operand: it vanished
            du = -1;
            return 0;
        }
        z = vmin;  // lead not determined inside the valid words
        stop = true;
    }
    if (z > room) {  // matrix capacity: shift only as far as it holds
        z = room;
        stop = true;
    }
    shift_left(u, z);
    du -= z;
    return z;
}

// One elimination: reduce u (the dividend) by v.  Fast path: the new lead is
// u[1] (z = 1), fetched by one shuffle while the window shifts by one.
// Returns z (the renormalisation shift); slow path handles z != 1, a vanished
// operand (du = -1) and an undetermined lead (stop).  hu1 tracks u's second
// coefficient (MODE 0: the fused pairs need it).
template <int MODE>
__device__ __forceinline__ int chain_step(uint32_t (&u)[GE], const uint32_t (&v)[GE],
                                          uint32_t& hu, uint32_t& hu1, uint32_t hv, int& du,
                                          int vj, int sup, int aged, bool& slow, bool& stop,
                                          Fld f) {
    using A = Arith<MODE>;
    const uint32_t p = f.p, x = hu, nx = A::neg(x, p);
#pragma unroll
    for (int e = 0; e < GE; ++e) u[e] = A::comb(hv, u[e], nx, v[e], f);
    const uint32_t h1 = from_lane(u[0], 1);
    const uint32_t h2 = MODE == 0 ? from_lane(u[0], 2) : 0u;
    if (A::nz(h1, p)) {
        shift_left1(u, GE);
        hu = h1;
        hu1 = h2;
        du -= 1;
        return 1;
    }
    slow = true;
    // bounds aged by the `aged` fast steps taken since they were refreshed
    const int vmin = vj < BIG ? vj - aged : BIG;
    const int room = PL - 1 - (sup + aged);
    const int z = renorm<MODE>(u, du, vmin, room, stop, p);
    hu = bcast(u[0]);
    if (MODE == 0) hu1 = from_lane(u[0], 1);
    return z;
}

// Two eliminations of u by v at once (MODE 0; deg u = deg v + 1 and the
// first step's new lead cc = (v0*u1 - u0*v1) * 2^-32 nonzero, so the second
// step reduces u again at equal degree): u1 = (v0*u - u0*X*v)/R, then
// u2 = (v0*u1 - cc*v)/R = (alpha*u + beta*X*v + gamma*v)/R with alpha = v0^2/R,
// beta = -u0*v0/R, gamma = -cc; top-aligned u2[t] = alpha*u[t+2] +
// beta*v[t+2] + gamma*v[t+1].  One 3-term reduction per word and one lead
// broadcast per two steps.  Returns the total shift z >= 2.
__device__ __forceinline__ int fused_step(uint32_t (&u)[GE], const uint32_t (&v)[GE], uint32_t& hu,
                                          uint32_t& hu1, uint32_t hv, uint32_t cc, int& du,
                                          int vj, int sup, int aged, bool& slow, bool& stop,
                                          Fld f, uint32_t& al, uint32_t& be, uint32_t& ga) {
    using A = Arith<0>;
    const uint32_t p = f.p;
    uint32_t us2[GE], vs2[GE], vs1[GE];
    shl_copy<2>(u, us2);
    shl_copy<2>(v, vs2);
    shl_copy<1>(v, vs1);
    al = A::mont(hv, hv, f);
    be = A::mont(hv, A::neg(hu, p), f);
    ga = A::canon(A::neg(cc, p), p);
#pragma unroll
    for (int e = 0; e < GE; ++e) u[e] = A::comb3(al, us2[e], be, vs2[e], ga, vs1[e], f);
    const uint32_t n0 = bcast(u[0]), n1 = from_lane(u[0], 1);
    if (A::nz(n0, p)) {
        hu = n0;
        hu1 = n1;
        du -= 2;
        return 2;
    }
    slow = true;
    const int vmin = vj < BIG ? vj - aged - 2 : BIG;
    const int room = PL - 1 - (sup + aged + 2);
    du -= 2;
    int z = 0;
    if (room > 0 && vmin > 0) {
        z = renorm<0>(u, du, vmin, room, stop, p);
    } else {
        stop = true;  // no room left past the pair: end the batch here
    }
    hu = bcast(u[0]);
    hu1 = from_lane(u[0], 1);
    return 2 + z;
}

// The fused pair as the steady state's fast path: everything is computed
// speculatively (the shifted copies before the scalars are known) and kept
// only if both cc and the new lead are nonzero; otherwise u is untouched and
// the general path takes over.
__device__ __forceinline__ bool fused_fast(uint32_t (&u)[GE], const uint32_t (&v)[GE], uint32_t& hu,
                                           uint32_t& hu1, uint32_t hv, uint32_t hv1, Fld f,
                                           uint32_t& al, uint32_t& be, uint32_t& ga) {
    using A = Arith<0>;
    const uint32_t p = f.p;
    uint32_t us2[GE], vs2[GE], vs1[GE], nu[GE];
    shl_copy<2>(u, us2);
    shl_copy<2>(v, vs2);
    shl_copy<1>(v, vs1);
    const uint32_t nx = A::neg(hu, p);
    const uint32_t cc = A::comb(hv, hu1, nx, hv1, f);
    al = A::mont(hv, hv, f);
    be = A::mont(hv, nx, f);
    ga = A::canon(A::neg(cc, p), p);
#pragma unroll
    for (int e = 0; e < GE; ++e) nu[e] = A::comb3(al, us2[e], be, vs2[e], ga, vs1[e], f);
    const uint32_t n0 = bcast(nu[0]), n1 = from_lane(nu[0], 1);
    if (!(A::nz(cc, p) && A::nz(n0, p))) return false;
#pragma unroll
    for (int e = 0; e < GE; ++e) u[e] = nu[e];
    hu = n0;
    hu1 = n1;
    return true;
}

// The fused pair as the steady state's fast path, with scalar lookahead: the
// new leads u'0 = (alpha*u2 + beta*v2 + gamma*v1)/R and u'1 (the same one
// word down) are computed as scalars from the operands' broadcast words 0..3,
// so the critical path is cc -> gamma -> one 3-term reduction; the vector
// update and the broadcast of u'2, u'3 (needed two pairs later as the
// dividend's, one pair later as the divisor's) run off it.  Everything is
// speculative and kept only if cc and u'0 are nonzero; otherwise u and its
// words are untouched and the general path takes over.
__device__ __forceinline__ bool fused_la(uint32_t (&u)[GE], const uint32_t (&v)[GE], uint32_t& u0,
                                         uint32_t& u1, uint32_t& u2, uint32_t& u3, uint32_t v0,
                                         uint32_t v1, uint32_t v2, uint32_t v3, Fld f,
                                         uint32_t& al, uint32_t& be, uint32_t& ga) {
    using A = Arith<0>;
    const uint32_t p = f.p;
    uint32_t us2[GE], vs2[GE], vs1[GE], nu[GE];
    shl_copy<2>(u, us2);
    shl_copy<2>(v, vs2);
    shl_copy<1>(v, vs1);
    const uint32_t nx = A::neg(u0, p);
    const uint32_t cc = A::comb(v0, u1, nx, v1, f);
    al = A::mont(v0, v0, f);
    be = A::mont(v0, nx, f);
    ga = A::canon(A::neg(cc, p), p);
    const uint32_t n0 = A::comb3(al, u2, be, v2, ga, v1, f);
    const uint32_t n1 = A::comb3(al, u3, be, v3, ga, v2, f);
#pragma unroll
    for (int e = 0; e < GE; ++e) nu[e] = A::comb3(al, us2[e], be, vs2[e], ga, vs1[e], f);
    if (!(A::nz(cc, p) && A::nz(n0, p))) return false;
#pragma unroll
    for (int e = 0; e < GE; ++e) u[e] = nu[e];
    u0 = n0;
    u1 = n1;
    u2 = from_lane(nu[0], 2);
    u3 = from_lane(nu[0], 3);
    return true;
}

// Two fused pairs back to back (u by v, then v by the new u) as one
// branch-free block: the four nonzero conditions are checked once at the end
// and nothing is committed unless all hold, so the scheduler can interleave
// the second pair's scalar chain with the first pair's vector update (in-order
// issue would otherwise stall the second chain behind the first's shuffles).
struct PairOut {
    uint32_t al1, be1, ga1, al2, be2, ga2;
};
__device__ __forceinline__ bool fused_pair_la(uint32_t (&u)[GE], uint32_t (&v)[GE], uint32_t& u0,
                                              uint32_t& u1, uint32_t& u2, uint32_t& u3,
                                              uint32_t& v0, uint32_t& v1, uint32_t& v2,
                                              uint32_t& v3, Fld f, PairOut& o) {
    using A = Arith<0>;
    const uint32_t p = f.p;
    uint32_t us2[GE], vs2[GE], vs1[GE], nu[GE], nus2[GE], nus1[GE], nv[GE];
    shl_copy<2>(u, us2);
    shl_copy<2>(v, vs2);
    shl_copy<1>(v, vs1);
    // pair 1: u <- u - (q1 X + q0) v
    const uint32_t nx = A::neg(u0, p);
    const uint32_t cc1 = A::comb(v0, u1, nx, v1, f);
    const uint32_t al1 = A::mont(v0, v0, f), be1 = A::mont(v0, nx, f);
    const uint32_t ga1 = A::canon(A::neg(cc1, p), p);
    const uint32_t n0 = A::comb3(al1, u2, be1, v2, ga1, v1, f);
    const uint32_t n1 = A::comb3(al1, u3, be1, v3, ga1, v2, f);
#pragma unroll
    for (int e = 0; e < GE; ++e) nu[e] = A::comb3(al1, us2[e], be1, vs2[e], ga1, vs1[e], f);
    const uint32_t n2 = from_lane(nu[0], 2), n3 = from_lane(nu[0], 3);
    shl_copy<2>(nu, nus2);
    shl_copy<1>(nu, nus1);
    // pair 2: v <- v - (r1 X + r0) u'
    const uint32_t ny = A::neg(v0, p);
    const uint32_t cc2 = A::comb(n0, v1, ny, n1, f);
    const uint32_t al2 = A::mont(n0, n0, f), be2 = A::mont(n0, ny, f);
    const uint32_t ga2 = A::canon(A::neg(cc2, p), p);
    const uint32_t m0 = A::comb3(al2, v2, be2, n2, ga2, n1, f);
    const uint32_t m1 = A::comb3(al2, v3, be2, n3, ga2, n2, f);
#pragma unroll
    for (int e = 0; e < GE; ++e) nv[e] = A::comb3(al2, vs2[e], be2, nus2[e], ga2, nus1[e], f);
    const uint32_t m2 = from_lane(nv[0], 2), m3 = from_lane(nv[0], 3);
    if (!(A::nz(cc1, p) & A::nz(n0, p) & A::nz(cc2, p) & A::nz(m0, p))) return false;
#pragma unroll
    for (int e = 0; e < GE; ++e) {
        u[e] = nu[e];
        v[e] = nv[e];
    }
    u0 = n0, u1 = n1, u2 = n2, u3 = n3;
    v0 = m0, v1 = m1, v2 = m2, v3 = m3;
    o = PairOut{al1, be1, ga1, al2, be2, ga2};
    return true;
}

// Warp 0 of CTA 0: the elimination chain of one batch on two fixed windows
// (wa for A, wb for B; a warp-uniform branch picks the dividend, no swaps).
// Capacity is checked through a step budget F: each fast step lowers the
// windows' joint validity and raises the matrix support by at most one, so
// the bounds are refreshed (pessimistically) only when F runs out or after a
// slow step.  Role rule, termination: oracle.cpp:58-66, 74-75; gcd.cpp:191-199.
template <int MODE>
__device__ void run_chain(BatchMeta& c, StepLog* log, volatile int* done, int jb, int M, Fld f,
                          const uint32_t* winA, const uint32_t* winB) {
    const unsigned par = batch_tag(jb);
    using A = Arith<MODE>;
    const uint32_t p = f.p;
    const int lane = threadIdx.x & 31;
    int da = int(c.da1), db = int(c.db1);  // exact: the windows start at the leads
    uint32_t wa[GE], wb[GE];
#pragma unroll
    for (int e = 0; e < GE; ++e) {
        wa[e] = winA[e * 32 + lane];
        wb[e] = winB[e * 32 + lane];
    }
    const int da0 = da, db0 = db;
    uint32_t ha = bcast(wa[0]), hb = bcast(wb[0]);
    uint32_t ha1 = from_lane(wa[0], 1), hb1 = from_lane(wb[0], 1);
    // joint validity: valid words of either window from the top (pessimistic);
    // BIG only while both windows hold their whole operands
    int vj = (da < W1 && db < W1) ? BIG : W1;
    int sup = 0;  // max matrix support (pessimistic)
    int dividend_a = c.dividend_a;
    const int cap = min(M, LOGCAP);
    const unsigned lb = log_base(log);
    int steps = 0, n = 0, term = 0, F = 0, F0 = 0;
    for (;;) {
        // oracle role rule: reduce the dividend while deg(dividend) >= deg(divisor)
        if (dividend_a) {
            if (da >= 0 && db >= 0 && da < db) dividend_a = 0;
        } else {
            if (da >= 0 && db >= 0 && db < da) dividend_a = 1;
        }
        if (F <= 0) {
            // refresh the pessimistic bounds with the F0 fast steps just taken
            if (vj < BIG) vj -= F0;
            sup += F0;
            F0 = 0;
            if (da < 0) { term = 1; break; }  // A vanished: gcd = B
            if (db < 0) { term = 2; break; }  // B vanished: gcd = A
            F = min(cap - steps, min(vj - 2, PL - 2 - sup));
            if (F <= 0) break;  // batch length, window or matrix exhausted
            F0 = F;
        }
        if (MODE == 0) {
            // steady state: degree-1 quotients, roles alternating every pair;
            // straight-line A-then-B pairs (a taken branch costs ~20 cycles).
            // Words 2, 3 of both windows as scalars for the lookahead (F >= 4
            // keeps at least 6 valid words).
            uint32_t al, be, ga;
#if GCD_CHAIN_LA == 0
            if (!dividend_a && F >= 2 && db == da + 1 && da >= 1 &&
                fused_fast(wb, wa, hb, hb1, ha, ha1, f, al, be, ga)) {  // align to A
                db -= 2;
                F -= 2;
                steps += 2;
                log_entry(lb, n++, par, al, be, ga, LOG_FUSED | 2u);
                dividend_a = 1;
            }
            if (dividend_a) {
                while (F >= 4 && da == db + 1 && db >= 2) {
                    if (!fused_fast(wa, wb, ha, ha1, hb, hb1, f, al, be, ga)) break;
                    da -= 2;
                    F -= 2;
                    steps += 2;
                    log_entry(lb, n++, par, al, be, ga, LOG_FUSED | LOG_UA | 2u);
                    dividend_a = 0;  // now db == da + 1, da >= 1
                    if (!fused_fast(wb, wa, hb, hb1, ha, ha1, f, al, be, ga)) break;
                    db -= 2;
                    F -= 2;
                    steps += 2;
                    log_entry(lb, n++, par, al, be, ga, LOG_FUSED | 2u);
                    dividend_a = 1;
                }
            }
#else
            if (F >= 4 && (dividend_a ? da == db + 1 && db >= 2 : db == da + 1 && da >= 2)) {
                uint32_t ha2 = from_lane(wa[0], 2), ha3 = from_lane(wa[0], 3);
                uint32_t hb2 = from_lane(wb[0], 2), hb3 = from_lane(wb[0], 3);
                if (!dividend_a &&
                    fused_la(wb, wa, hb, hb1, hb2, hb3, ha, ha1, ha2, ha3, f, al, be, ga)) {
                    db -= 2;  // align to A
                    F -= 2;
                    steps += 2;
                    log_entry(lb, n++, par, al, be, ga, LOG_FUSED | 2u);
                    dividend_a = 1;
                }
                if (dividend_a) {
                    // whole A-then-B rounds (F >= 4 also covers the second pair's
                    // lookahead words).  A failed round commits nothing:
                    // the general path below retakes its first pair.
                    PairOut o;
                    while (F >= 4 && da == db + 1 && db >= 2 &&
                           fused_pair_la(wa, wb, ha, ha1, ha2, ha3, hb, hb1, hb2, hb3, f, o)) {
                        log_entry(lb, n, par, o.al1, o.be1, o.ga1, LOG_FUSED | LOG_UA | 2u);
                        log_entry(lb, n + 1, par, o.al2, o.be2, o.ga2, LOG_FUSED | 2u);
                        n += 2;
                        da -= 2;
                        db -= 2;
                        F -= 4;
                        steps += 4;
                    }
                }
            }
#endif
            if (F <= 0) continue;  // refresh first
        }
        const int du = dividend_a ? da : db, dv = dividend_a ? db : da;
        if (dv == 0) { term = 3; break; }  // constant divisor: unit gcd
        const int aged = F0 - F;  // fast steps since the bounds were refreshed
        bool slow = false, stop = false;
        int z;
        if (MODE == 0 && F >= 2 && du == dv + 1) {
            // a degree-1 quotient: fuse its two steps unless the first one
            // drops the degree by more than one (cc = 0)
            const uint32_t u0 = dividend_a ? ha : hb, u1 = dividend_a ? ha1 : hb1;
            const uint32_t v0 = dividend_a ? hb : ha, v1 = dividend_a ? hb1 : ha1;
            const uint32_t cc = A::comb(v0, u1, A::neg(u0, p), v1, f);
            if (A::nz(cc, p)) {
                uint32_t al, be, ga;
                if (dividend_a)
                    z = fused_step(wa, wb, ha, ha1, hb, cc, da, vj, sup, aged, slow, stop, f, al,
                                   be, ga);
                else
                    z = fused_step(wb, wa, hb, hb1, ha, cc, db, vj, sup, aged, slow, stop, f, al,
                                   be, ga);
                F -= 2;
                if (slow) {
                    const int used = F0 - F - 2;
                    if (vj < BIG) vj -= used + z;
                    sup += used + z;
                    F = 0;
                    F0 = 0;
                }
                log_entry(lb, n++, par, al, be, ga,
                          LOG_FUSED | (dividend_a ? LOG_UA : 0u) | unsigned(z));
                steps += 2;
                if (stop) break;
                continue;
            }
        }
        const uint32_t x = dividend_a ? ha : hb, y = dividend_a ? hb : ha;
        if (dividend_a)
            z = chain_step<MODE>(wa, wb, ha, ha1, hb, da, vj, sup, aged, slow, stop, f);
        else
            z = chain_step<MODE>(wb, wa, hb, hb1, ha, db, vj, sup, aged, slow, stop, f);
        --F;
        if (slow) {  // exact bookkeeping for this step, then re-derive the budget
            const int used = F0 - F - 1;  // fast steps before this one
            if (vj < BIG) vj -= used + z;
            sup += used + z;
            F = 0;
            F0 = 0;
        }
        log_entry(lb, n++, par, x, y, 0u, (dividend_a ? LOG_UA : 0u) | unsigned(z));
        ++steps;
        if (stop) break;
    }
    if (lane == 0) {
        c.da0 = da0;
        c.db0 = db0;
        c.da1 = da;
        c.db1 = db;
        c.steps = steps;
        c.term = term;
        c.dividend_a = dividend_a;
        c.sa = da0 - (da < 0 ? da0 : da);  // top moves (unused for a vanished row)
        c.sb = db0 - (db < 0 ? db0 : db);
        st_release_cta(done, int((par << 10) | unsigned(n + 1)));  // batch tag | entry count + 1
    }
}

// One log entry applied to a matrix row: u (the dividend's row) from u, v.
// Fused pair with no extra shift (the steady state): straight-line.
__device__ __forceinline__ void replay_fused2(uint32_t (&u)[PE], const uint32_t (&v)[PE],
                                              const uint4& en, Fld f) {
    uint32_t us2[PE], vs2[PE], vs1[PE];
    shr_copy<2>(u, us2);
    shr_copy<2>(v, vs2);
    shr_copy<1>(v, vs1);
#pragma unroll
    for (int e = 0; e < PE; ++e) u[e] = Arith<0>::comb3(en.x, us2[e], en.y, vs2[e], en.z, vs1[e], f);
}

template <int MODE>
__device__ __forceinline__ void replay_entry(uint32_t (&u)[PE], const uint32_t (&v)[PE],
                                             const uint4& en, Fld f) {
    using A = Arith<MODE>;
    const int z = int(en.w & LOG_Z);
    if (MODE == 0 && (en.w & LOG_FUSED)) {
        // Pu[e] <- alpha*Pu[e-2] + beta*Pv[e-2] + gamma*Pv[e-1], then >> z-2
        uint32_t us2[PE], vs2[PE], vs1[PE];
        shr_copy<2>(u, us2);
        shr_copy<2>(v, vs2);
        shr_copy<1>(v, vs1);
#pragma unroll
        for (int e = 0; e < PE; ++e)
            u[e] = Arith<0>::comb3(en.x, us2[e], en.y, vs2[e], en.z, vs1[e], f);
        if (z > 2) shift_right(u, z - 2);
    } else {
        const uint32_t nx = A::neg(en.x, f.p);
#pragma unroll
        for (int e = 0; e < PE; ++e) u[e] = A::comb(en.y, u[e], nx, v[e], f);
        if (z == 1) shift_right1(u, PE);
        else shift_right(u, z);
    }
}

// Warps 1 and 2 of CTA 0: replay the step log into matrix column `col` (row
// A in ra, row B in rb: fixed registers, a uniform branch picks the row the
// entry reduces); the next entry is fetched while one is applied.  Then
// publish the column (canonical) to Pg and Ps.
template <int MODE>
__device__ void run_replay(int col, const StepLog* log, volatile int* done, int jb, Fld f,
                           uint64_t* rec, unsigned rtag, uint32_t* Ps, int* hi_out,
                           volatile int* ring_ok, long long* tex = nullptr) {
    const unsigned par = batch_tag(jb);
    // the chain finished this batch with fewer than i + 1 entries
    // A plain (volatile) read: `done` only bounds the entry count, and every
    // entry carries its own tag.  The shared address is converted once (the
    // conversion reads SR_CgaCtaId, slow, and this runs in the polling loop).
    const unsigned done_sa = static_cast<unsigned>(__cvta_generic_to_shared(const_cast<int*>(done)));
    auto ended = [&](int i) {
        unsigned d;
        asm volatile("ld.volatile.shared::cta.u32 %0, [%1];" : "=r"(d) : "r"(done_sa));
        return (d >> 10) == par && int(d & 0x3FFu) - 1 <= i;
    };
    using A = Arith<MODE>;
    const uint32_t p = f.p;
    const int lane = threadIdx.x & 31;
    uint32_t ra[PE], rb[PE];
#pragma unroll
    for (int e = 0; e < PE; ++e) ra[e] = rb[e] = 0u;
    if (lane == 0) {  // identity: row A col 0 = 1, row B col 1 = 1
        if (col == 0) ra[0] = 1u;
        else rb[0] = 1u;
    }
    int ha = col == 0 ? 0 : -1, hb = col == 0 ? -1 : 0;  // support bounds
    constexpr unsigned KIND = LOG_FUSED | LOG_UA | LOG_Z;
    const unsigned lb = log_base(log);
    const int last = LOGCAP - 1;
    int i = 0;
#if GCD_REPLAY_SIMPLE == 2
    // One poll loop for the next pair (A then B entry, the steady state) with
    // the chain's end: the common path falls through (taken branches cost
    // tens of cycles here), and an ended chain leaves a single entry or none.
    for (;;) {
        uint4 en = log_get(lb, i), nx = log_get(lb, min(i + 1, last));
        unsigned d;
        for (;;) {
            asm volatile("ld.volatile.shared::cta.u32 %0, [%1];" : "=r"(d) : "r"(done_sa));
            const bool h0 = (en.w >> 10) == par, h1 = (nx.w >> 10) == par;
            const int cnt = (d >> 10) == par ? int(d & 0x3FFu) - 1 : 1 << 20;  // entries, once ended
            if ((h0 && h1) || (h0 && cnt <= i + 1) || cnt <= i) break;
            en = log_get(lb, i);
            nx = log_get(lb, min(i + 1, last));
        }
        const bool h0 = (en.w >> 10) == par, h1 = (nx.w >> 10) == par;
        if (!h0) break;  // the chain ended before entry i
        if (MODE == 0 && h1 && (en.w & KIND) == (LOG_FUSED | LOG_UA | 2u) &&
            (nx.w & KIND) == (LOG_FUSED | 2u)) {
            replay_fused2(ra, rb, en, f);
            replay_fused2(rb, ra, nx, f);
            const int h1s = max(ha, hb) >= 0 ? max(ha, hb) + 2 : -1;
            ha = h1s;
            hb = h1s >= 0 ? max(h1s, hb) + 2 : -1;
            i += 2;
            continue;
        }
        const int z = int(en.w & LOG_Z), hmax = max(ha, hb);
        if (en.w & LOG_UA) {
            replay_entry<MODE>(ra, rb, en, f);
            ha = hmax >= 0 ? hmax + z : -1;
        } else {
            replay_entry<MODE>(rb, ra, en, f);
            hb = hmax >= 0 ? hmax + z : -1;
        }
        ++i;
    }
#elif GCD_REPLAY_SIMPLE
    // One entry at a time: poll it, fetch the next one, apply.  (Entries
    // arrive every ~270 cycles and apply in ~180: the replay waits on the
    // chain, so what matters is how soon it notices an entry, not batching.)
    uint4 en = log_get(lb, 0);
    for (;;) {
        bool fin = false;
        while ((en.w >> 10) != log_seq(i, par)) {
            if (ended(i)) {
                fin = true;
                break;
            }
            en = log_get(lb, i);
        }
        if (fin) break;
        const uint4 nx = log_get(lb, min(i + 1, last));
        const int z = int(en.w & LOG_Z), hmax = max(ha, hb);
        const unsigned kind = en.w & KIND;
        if (en.w & LOG_UA) {
            if (MODE == 0 && kind == (LOG_FUSED | LOG_UA | 2u)) replay_fused2(ra, rb, en, f);
            else replay_entry<MODE>(ra, rb, en, f);
            ha = hmax >= 0 ? hmax + z : -1;
        } else {
            if (MODE == 0 && kind == (LOG_FUSED | 2u)) replay_fused2(rb, ra, en, f);
            else replay_entry<MODE>(rb, ra, en, f);
            hb = hmax >= 0 ? hmax + z : -1;
        }
        ++i;
        en = nx;
    }
#else
    uint4 en = log_get(lb, 0), nx = log_get(lb, 1);
    for (;;) {
        if (MODE == 0) {
            // steady state: published A pair then B pair, applied straight-line
            // with the next two entries already in flight (one taken branch)
            while ((en.w >> 10) == log_seq(i, par) && (nx.w >> 10) == log_seq(i + 1, par) &&
                   (en.w & KIND) == (LOG_FUSED | LOG_UA | 2u) &&
                   (nx.w & KIND) == (LOG_FUSED | 2u)) {
#ifdef GCD_TRACE
                if (col == 0 && lane == 0) g_tb[i] = clock64();
#endif
                const uint4 n2 = log_get(lb, min(i + 2, last)), n3 = log_get(lb, min(i + 3, last));
#ifdef GCD_TRACE
                if (col == 0 && lane == 0) g_tr[i] = clock64();
#endif
                replay_fused2(ra, rb, en, f);
                replay_fused2(rb, ra, nx, f);
                const int h1 = max(ha, hb) >= 0 ? max(ha, hb) + 2 : -1;
                ha = h1;
                hb = h1 >= 0 ? max(h1, hb) + 2 : -1;
                en = n2;
                nx = n3;
                i += 2;
            }
        }
        while ((en.w >> 10) != log_seq(i, par)) {
            if (ended(i)) break;
            en = log_get(lb, i);  // spin: warps 1-2 do not share the chain's SMSP
        }
        if ((en.w >> 10) != log_seq(i, par)) break;
#ifdef GCD_TRACE
        if (col == 0 && lane == 0) g_tp[i] = clock64();
#endif
        if (MODE == 0 && (en.w & KIND) == (LOG_FUSED | LOG_UA | 2u) &&
            (nx.w >> 10) != log_seq(i + 1, par)) {
            // a steady A pair whose partner is not yet published: wait for it
            while ((nx.w >> 10) != log_seq(i + 1, par)) {
                if (ended(i + 1)) break;
                nx = log_get(lb, min(i + 1, last));
            }
#ifdef GCD_TRACE
            if (col == 0 && lane == 0) g_ta[i] = clock64();
#endif
            if ((nx.w >> 10) == log_seq(i + 1, par) && (nx.w & KIND) == (LOG_FUSED | 2u)) continue;
        }
        const int z = int(en.w & LOG_Z), hmax = max(ha, hb);
#ifdef GCD_TRACE
        if (col == 0 && lane == 0) g_tr[i] = clock64();
#endif
        if (en.w & LOG_UA) {
            replay_entry<MODE>(ra, rb, en, f);
            ha = hmax >= 0 ? hmax + z : -1;
        } else {
            replay_entry<MODE>(rb, ra, en, f);
            hb = hmax >= 0 ? hmax + z : -1;
        }
        ++i;
        en = (nx.w >> 10) == log_seq(i, par) ? nx : log_get(lb, min(i, last));
        nx = log_get(lb, min(i + 1, last));
    }
#endif
    if (tex && lane == 0) *tex = clock64();
    while (ld_acquire_cta(ring_ok) < jb) {
    }
    uint64_t* Pa = rec + (0 * 2 + col) * PL;  // row A, column col
    uint64_t* Pb = rec + (1 * 2 + col) * PL;  // row B, column col
#pragma unroll
    for (int e = 0; e < PE; ++e) {
        const uint32_t va = A::canon(ra[e], p), vb = A::canon(rb[e], p);
        st_tag(Pa + e * 32 + lane, va, rtag);
        st_tag(Pb + e * 32 + lane, vb, rtag);
        // the window builder's copy, index-reversed (a correlation run as convolution)
        Ps[(0 * 2 + col) * PL + (PL - 1) - (e * 32 + lane)] = va;
        Ps[(1 * 2 + col) * PL + (PL - 1) - (e * 32 + lane)] = vb;
    }
    if (lane == 0) {
        hi_out[0 * 2 + col] = min(ha, PL - 1);
        hi_out[1 * 2 + col] = min(hb, PL - 1);
    }
}

}  // namespace

// ------------------------------------------------------- flags (gpu scope) --
// Warp-level: min over the bulk CTAs' progress words (all loads in flight).
constexpr int MAXBULK = 160;
__device__ __forceinline__ unsigned min_progress(const unsigned* prog, int nbulk) {
    const int lane = threadIdx.x & 31;
    unsigned v[MAXBULK / 32];
#pragma unroll
    for (int k = 0; k < MAXBULK / 32; ++k)
        v[k] = lane + 32 * k < nbulk ? ld_relaxed_gpu(prog + lane + 32 * k) : ~0u;
    unsigned mn = ~0u;
#pragma unroll
    for (int k = 0; k < MAXBULK / 32; ++k) mn = min(mn, v[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    return mn;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Thread 0 waits until *p >= target; the CTA then proceeds together.  A pure
// spin: one L2 round trip in flight per CTA, and no sleep wake-up delay.
__device__ __forceinline__ void cta_wait_ge(const unsigned* p, unsigned target) {
    if (threadIdx.x == 0) spin_until_geq(p, target);
    __syncthreads();
}

// Load the top W1 words of tagged state Z below `deg` into w; lower `deg` past
// zero words until w[0] is the nonzero lead (or deg = -1: zero operand).
// Warp-uniform.
template <int MODE>
__device__ void load_top(uint32_t (&w)[GE], const uint64_t* Z, unsigned tag, long long& deg,
                         uint32_t p) {
    const int lane = threadIdx.x & 31;
    while (deg >= 0) {
        uint64_t r[GE];
#pragma unroll
        for (int e = 0; e < GE; ++e) {
            const long long x = deg - (e * 32 + lane);
            r[e] = x >= 0 ? ld_rlx64(Z + x) : (uint64_t(tag) << 32);
        }
#pragma unroll
        for (int e = 0; e < GE; ++e) {
            const long long x = deg - (e * 32 + lane);
            w[e] = tag_resolve(Z + (x >= 0 ? x : 0), r[e], tag);
        }
        const int z = first_nz<MODE>(w, 0, p);
        if (z == 0) return;
        deg -= z < 0 ? W1 : z;
    }
}

// Warp-level: top-aligned W1-word window of Z at degree `deg` into smem; lowers
// `deg` past zero words until win[0] is the lead (deg = -1: zero operand).
template <int MODE>
__device__ void window_from_global(uint32_t* win, const uint64_t* Z, unsigned tag, long long& deg,
                                   uint32_t p) {
    uint32_t w[GE];
    load_top<MODE>(w, Z, tag, deg, p);
#pragma unroll
    for (int e = 0; e < GE; ++e) win[e * 32 + (threadIdx.x & 31)] = w[e];
    __syncwarp();
}


// Both next windows, top-aligned, from S_j's top region and the batch matrix:
//   winA[t] = sum_e Pa1[e] topA[t+e] + sum_e Pa2[e] topB[t+e]   (t < W1)
// and winB likewise with Pb1, Pb2.  Ps holds each polynomial index-reversed
// (Ps[c][PL-1-e] = P_c[e]), so with u = PL-1-e the sum is the convolution
// conv_accumulate computes.  Split-K over BUILD_PARTS parts (term x half of
// the support), one part per warp; the 32 lanes hold the 2 x W1/4 quads of
// 4 consecutive words (shared-memory reads: broadcast or consecutive, no
// bank conflicts), and the parts meet in a shared-memory reduction.
#ifndef GCD_BUILD_PARTS
#define GCD_BUILD_PARTS 4  // 8 (warp 7 builds, publishes after) measured 15 % slower
#endif
#ifndef GCD_PUB_FIRST
#define GCD_PUB_FIRST 1  // 8 parts: warp 7 publishes the meta words before its part
#endif
constexpr int BUILD_PARTS = GCD_BUILD_PARTS;
static_assert(2 * (W1 / 4) == 32, "window builder: one (window, quad) per lane");
static_assert(BUILD_PARTS <= GCD_T / 32, "window builder: one part per warp");
__device__ void build_window_part(int part, uint32_t* red, const uint32_t* Ps, const int* hi,
                                  const uint32_t* topA, const uint32_t* topB,
                                  const FieldParams& F) {
    constexpr int SPAN = 2 * PL / BUILD_PARTS;  // terms per part
    const int lane = threadIdx.x & 31, w = lane >> 4, q = lane & 15;
    const int term = part / (BUILD_PARTS / 2), u0 = (part % (BUILD_PARTS / 2)) * SPAN;
    const int c = 2 * w + term;  // Pa1, Pa2, Pb1, Pb2
    uint64_t acc[4] = {0, 0, 0, 0};
    uint32_t since = 0;
    // reversed support: u in [PL-1-hi, PL-1]
    if (hi[c] >= 0 && u0 + SPAN - 1 >= PL - 1 - hi[c]) {
        if (F.fold_terms >= SPAN)  // (every prime below 2^29): straight-line, no fold
            conv_accumulate_fixed<4, SPAN / 4>(acc, Ps + c * PL + u0, term ? topB : topA,
                                               4 * q + PL - 1 - u0);
        else
            conv_accumulate<4>(acc, Ps + c * PL + u0, SPAN / 4, term ? topB : topA,
                               4 * q + PL - 1 - u0, since, F);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) red[part * (2 * W1) + w * W1 + 4 * q + r] = reduce(acc[r], F);
}

// Named barrier over the first n threads' warps (n a multiple of 32).
__device__ __forceinline__ void bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// CTA 0: the sequential part.  Per batch j: chain (warp 0) || replay (warps
// 1-2) || prefetch of S_j's top region (warps 3-7); then warp 7 publishes
// the matrix (its fence waits for the stores to reach L2) while warps 0-6
// build the next windows from it.  Never waits for the bulk of the batch it
// just finished (only for the one before, which had a whole batch).
constexpr int BUILDERS = BUILD_PARTS == 8 ? GCD_T : GCD_T - 32;  // warps 0-6 (+7)
template <int MODE>
__device__ int head_cta(const GcdArgs& g, BatchMeta& ctl, StepLog* log, uint32_t* smem_rest,
                        volatile int* done, int* hi_s, int nbulk) {
    const FieldParams F = g.F;
    const int warp = threadIdx.x >> 5;
    uint32_t* winA = smem_rest;
    uint32_t* winB = winA + W1;
    uint32_t* topA = winB + W1;         // W1 + PL words
    uint32_t* topB = topA + W1 + PL;
    uint32_t* Ps = topB + W1 + PL;      // 4 * PL
    uint32_t* red = Ps + 4 * PL;        // BUILD_PARTS x 2 * W1 builder partials
    __shared__ long long da0s[2], db0s[2];  // batch start degrees, by batch parity
    __shared__ long long hst[12];  // MMM_GCD_STATS: accumulated here, flushed at the end
    __shared__ long long tpub_s, tex_s;
    __shared__ long long hx[4];
    if (threadIdx.x < 4) hx[threadIdx.x] = 0;
    __shared__ volatile int ring_ok;  // record slot of batch <= ring_ok is free
    __shared__ unsigned minprog_s;    // min bulk progress seen this batch
    if (threadIdx.x < 12) hst[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        tpub_s = 0;
        ring_ok = -1;
    }
    if (threadIdx.x == 0) *done = 0;
    for (int i = threadIdx.x; i < LOGCAP; i += GCD_T)  // no stale tags from earlier kernels
        reinterpret_cast<uint4*>(log)[i] = make_uint4(0u, 0u, 0u, 0u);
    if (warp == 0) {
        long long da = g.na - 1, db = g.nb - 1;
        window_from_global<MODE>(winA, g.XA[0], 1u, da, F.p);
        window_from_global<MODE>(winB, g.XB[0], 1u, db, F.p);
        if ((threadIdx.x & 31) == 0) {
            ctl.da1 = da;
            ctl.db1 = db;
            ctl.dividend_a = 1;  // oracle_gcd: x = a is the first dividend (oracle.cpp:70)
            da0s[0] = da;
            db0s[0] = db;
        }
    }
    __syncthreads();
    long long t0 = clock64();
    for (int j = 0;; ++j) {
        if (warp == 0) {
            run_chain<MODE>(ctl, log, done, j, g.M, Fld{F.p, F.pinv}, winA, winB);
            if (g.stats && threadIdx.x == 0) hst[4] += clock64() - t0;
        } else if (warp <= 2) {
            // (record slot j % RING is written at the end, once ring_ok says it is free)
            run_replay<MODE>(warp - 1, log, done, j, Fld{F.p, F.pinv}, g.rec + (j % RING) * REC_W,
                             unsigned(j + 1), Ps, hi_s, &ring_ok,
                             (g.stats && warp == 1) ? &tex_s : nullptr);
            if (g.stats && threadIdx.x == 32) {
                hst[5] += clock64() - t0;
                hst[9] += tex_s - t0;
            }
        } else {
            // Warp 3 prefetches S_j's top region: tagged words, each polled until
            // the bulk CTA that owns it wrote it for batch j - 1.  Only warps 3
            // and 7 (SMSP 3) work here: a polling warp on SMSPs 0-2 would take
            // issue slots from the chain (warp 0) or a replay warp (1, 2).
            if (warp == 3) {
                const long long da0 = da0s[j & 1], db0 = db0s[j & 1];  // ordered by bar 2
                const uint64_t* ZA = g.XA[j % NBUF];
                const uint64_t* ZB = g.XB[j % NBUF];
                const unsigned tg = unsigned(j + 1);
                constexpr int K = (W1 + PL) / 32;
                const int lane = threadIdx.x & 31;
                const uint64_t* ad[2 * K];
                uint64_t r[2 * K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const long long xa = da0 - (lane + 32 * k), xb = db0 - (lane + 32 * k);
                    ad[k] = ZA + (xa >= 0 ? xa : 0);
                    ad[K + k] = ZB + (xb >= 0 ? xb : 0);
                    r[k] = xa >= 0 ? ld_rlx64(ad[k]) : uint64_t(tg) << 32;
                    r[K + k] = xb >= 0 ? ld_rlx64(ad[K + k]) : uint64_t(tg) << 32;
                }
                tag_resolve_all<2 * K>(ad, r, tg);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    topA[lane + 32 * k] = uint32_t(r[k]);
                    topB[lane + 32 * k] = uint32_t(r[K + k]);
                }
                if (g.stats && j > 0 && lane == 0) {
                    hst[10] += gtimer() - tpub_s;
                    hst[11] += 1;
                }
            } else if (warp == 7) {
                // record slot j % RING is free once every bulk CTA finished batch
                // j - RING (the replay's matrix and warp 7's meta wait for this);
                // the minimum also travels in the record for the bulk's guard
                unsigned mn = min_progress(g.prog, nbulk);
                while (j >= RING && mn < unsigned(j - RING + 1)) mn = min_progress(g.prog, nbulk);
                if ((threadIdx.x & 31) == 0) {
                    minprog_s = mn;
                    st_release_cta(&ring_ok, j);
                }
            }
            if (g.stats && threadIdx.x == 96) hst[6] += clock64() - t0;
        }
        __syncthreads();
        if (g.stats && threadIdx.x == 0) hst[2] += clock64() - t0;
        BatchMeta m = ctl;
        m.da0 = da0s[j & 1];
        m.db0 = db0s[j & 1];
        for (int i = 0; i < 4; ++i) m.hi[i] = hi_s[i];
        m.err = (m.steps == 0 && m.term == 0) ? 1 : 0;
        const bool last = m.term || m.err;
        // warp 7 publishes batch j: the record's meta words (the replay wrote P)
        auto publish = [&]() {
            const int l = threadIdx.x - 224;
            // selects on registers (a runtime index into m would put it in local memory)
            const int h0 = m.hi[0], h1 = m.hi[1], h2 = m.hi[2], h3 = m.hi[3];
            int v = l == 0 ? int(m.da0) : l == 1 ? int(m.db0) : l == 2 ? int(m.da1)
                  : l == 3 ? int(m.db1) : l == 4 ? m.steps : l == 5 ? m.term
                  : l == 6 ? m.dividend_a : l == 7 ? m.err : l == 8 ? m.sa
                  : l == 9 ? m.sb : l == 10 ? h0 : l == 11 ? h1 : l == 12 ? h2 : h3;
            long long tp = g.stats ? gtimer() : 0;
            tp = __shfl_sync(0xffffffffu, tp, 0);
            if (l == 14) v = int(uint32_t(tp));
            if (l == 15) v = int(uint32_t(uint64_t(tp) >> 32));
            if (l == 16) v = int(minprog_s);
            if (l < META_W)
                st_tag(g.rec + (j % RING) * REC_W + 4 * PL + l, uint32_t(v), unsigned(j + 1));
            if (threadIdx.x == 224 && g.stats) {
                tpub_s = tp;
                hst[0] += 1;
                hst[1] += m.steps;
            }
        };
        if (last) {
            if (warp == 7) publish();
            __syncthreads();  // hst complete
            if (g.stats && threadIdx.x == 224) {
                for (int i = 0; i < 10; ++i) g.stats[i == 7 ? 8 : (i == 8 ? 9 : (i == 9 ? 10 : i))] = hst[i];
                g.stats[17] = hst[10];
                for (int i = 0; i < 4; ++i) g.stats[21 + i] = hx[i];
                g.stats[19] = hst[11];
            }
            return j;
        }
        if (warp == 7 && BUILD_PARTS < 8) {  // publish now; the next batch's prefetch group
            publish();
            continue;
        }
        // next windows, top-aligned, from S_j and the batch matrix (with 8
        // parts warp 7 builds first and publishes after: the bulk has slack)
        if (g.stats && threadIdx.x == 0) hx[0] += clock64() - t0;
        if (BUILD_PARTS == 8 && GCD_PUB_FIRST && warp == 7) publish();
        if (warp < BUILD_PARTS) build_window_part(warp, red, Ps, hi_s, topA, topB, F);
        if (g.stats && threadIdx.x == 0) hx[1] += clock64() - t0;
        if (BUILD_PARTS == 8 && !GCD_PUB_FIRST && warp == 7) publish();
        if (g.stats && (g.dbg & 4)) {  // timing experiment: the same part again (warm)
            if (warp < BUILD_PARTS) build_window_part(warp, red, Ps, hi_s, topA, topB, F);
            if (threadIdx.x == 0) hx[3] += clock64() - t0;
        }
        bar_sync(2, BUILDERS);
        // sum the parts (winA then winB); a new lead that is zero means the bound
        // after the batch is not the lead (degree dropped past the valid words)
        bool stale = false;
        if (threadIdx.x < 2 * W1) {
            uint64_t sum = 0;
#pragma unroll
            for (int pt = 0; pt < BUILD_PARTS; ++pt) sum += red[pt * (2 * W1) + threadIdx.x];
            const uint32_t v = reduce(sum, F);
            (threadIdx.x < W1 ? winA : winB)[threadIdx.x & (W1 - 1)] = v;
            stale = v == 0u && ((threadIdx.x == 0 && m.da1 >= 0) || (threadIdx.x == W1 && m.db1 >= 0));
        }
        if (threadIdx.x == 0) {
            da0s[(j + 1) & 1] = m.da1;  // read by the prefetch after the barrier below
            db0s[(j + 1) & 1] = m.db1;
        }
        if (g.stats && threadIdx.x == 0) hst[7] += clock64() - t0;
        // one barrier: the windows and da0s/db0s, and whether a lead is stale
        int fb;
        asm volatile(
            "{ .reg .pred p, q; setp.ne.u32 p, %1, 0; bar.red.or.pred q, 2, %2, p; selp.s32 %0, 1, 0, q; }"
            : "=r"(fb) : "r"(int(stale)), "r"(BUILDERS) : "memory");
        if (g.stats && threadIdx.x == 0) hst[8] += clock64() - t0;
        if (fb) {  // take the exact state from the bulk instead
            if (warp == 0) {  // tagged reads wait for the bulk's batch j
                long long da = m.da1, db = m.db1;
                window_from_global<MODE>(winA, g.XA[(j + 1) % NBUF], unsigned(j + 2), da, F.p);
                window_from_global<MODE>(winB, g.XB[(j + 1) % NBUF], unsigned(j + 2), db, F.p);
                if ((threadIdx.x & 31) == 0) {
                    ctl.da1 = da;
                    ctl.db1 = db;
                    da0s[(j + 1) & 1] = da;
                    db0s[(j + 1) & 1] = db;
                }
            }
            bar_sync(2, BUILDERS);
        }
        if (g.stats && threadIdx.x == 0) hx[2] += clock64() - t0;
        if (unsigned(j + 1) % TAG_MASK == 0u) {  // tag wraps (2^22 batches): clear the log
            for (int i = threadIdx.x; i < LOGCAP; i += BUILDERS)
                reinterpret_cast<uint4*>(log)[i] = make_uint4(0u, 0u, 0u, 0u);
            bar_sync(2, BUILDERS);
        }
        if (g.stats && threadIdx.x == 0) {
            const long long t1 = clock64();
            hst[3] += t1 - t0;
            t0 = t1;
        }
        if (g.stats) t0 = clock64();
    }
}

// Bulk apply of one batch matrix to this CTA's outputs [s0, s1) of the new
// state (row A: indices < na1, then row B):
//   out[x] = sum_e P1[e] Z1[x + s1 - e] + sum_e P2[e] Z2[x + s2 - e].
// Per pass of up to APPLY_OUT outputs, P and the four operand windows the
// pass needs are staged with one L2 round trip; a work item is (4 consecutive
// outputs, one quarter of the MAC range: term x half of the support), run by
// the register-tiled conv_accumulate<4>, and the 4 quarters (adjacent lanes)
// meet in a two-level butterfly.  (gcd.cpp:252-300 UpdateMatrix apply.)
constexpr int APPLY_OUT = GCD_T;  // outputs per pass: one work item per thread
#ifndef GCD_OUT_PER_CTA
#define GCD_OUT_PER_CTA 128  // target outputs per bulk CTA (grid size)
#endif
constexpr int APPLY_WORDS = 4 * PL + 2 * (APPLY_OUT + 8) + 4 * (PL + 4);

static_assert(APPLY_OUT + PL + 4 <= 2 * GCD_T, "apply: two staged words per thread and window");
static_assert(4 * PL == GCD_T, "apply: one matrix word per thread");
__device__ void apply_batch(const GcdArgs& g, const BatchMeta& m, int j, long long s0, long long s1,
                            uint32_t* sm, const uint64_t* rec, long long* ph) {
    const long long tb = ph ? clock64() : 0;
    const FieldParams F = g.F;
    const int tid = threadIdx.x;
    uint32_t* P = sm;  // Pa1, Pa2, Pb1, Pb2: the record's matrix, staged with the first pass
    uint32_t* Wb = sm + 4 * PL;
    const uint64_t* Z[2] = {g.XA[j % NBUF], g.XB[j % NBUF]};
    const unsigned tg = unsigned(j + 1);  // S_j in, S_{j+1} out
    const long long deg[2] = {m.da0, m.db0};
    uint64_t* out[2] = {g.XA[(j + 1) % NBUF], g.XB[(j + 1) % NBUF]};
    const long long na1 = m.da1 + 1 > 0 ? m.da1 + 1 : 0;
    // shift of term t for row r: Z_t index = x + sh[2r + t] - e
    const long long sh[4] = {m.sa, m.sa + m.db0 - m.da0, m.sb + m.da0 - m.db0, m.sb};
    for (long long c0 = s0; c0 < s1; c0 += APPLY_OUT) {
        const long long c1 = min(c0 + APPLY_OUT, s1);
        const long long xs[2] = {min(c0, na1), max(c0 - na1, 0LL)};
        const int n[2] = {int(min(c1, na1) - xs[0]), int(max(c1 - na1, 0LL) - xs[1])};
        const int qn[2] = {(n[0] + 3) >> 2, (n[1] + 3) >> 2};
        const int L[2] = {4 * qn[0] + PL + 4, 4 * qn[1] + PL + 4};
        uint32_t* W[4] = {Wb, Wb + L[0], Wb + 2 * L[0], Wb + 2 * L[0] + L[1]};
        __syncthreads();  // previous pass done with the windows
        if (ph && c0 == s0) ph[0] += clock64() - tb;
        // W[2r + t][y] = Z_t[xs_r + sh - (PL - 1) + y], zero outside [0, deg_t]:
        // all loads in flight first, then each polled until tagged S_j
        // (slot 8: this thread's matrix word, first pass only)
        const uint64_t* ad[9];
        uint64_t rw[9];
        unsigned live = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int r = w >> 1, t = w & 1;
            const long long base = xs[r] + sh[w] - (PL - 1);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int y = tid + k * GCD_T;
                const long long x = base + y;
                const bool lv = y < L[r] && n[r] > 0 && x >= 0 && x <= deg[t];
                ad[2 * w + k] = Z[t] + (lv ? x : 0);
                rw[2 * w + k] = lv ? ld_rlx64(ad[2 * w + k]) : uint64_t(tg) << 32;
                live |= lv ? 1u << (2 * w + k) : 0u;
            }
        }
        ad[8] = rec + tid;
        rw[8] = c0 == s0 ? ld_rlx64(ad[8]) : uint64_t(tg) << 32;
        tag_resolve_all<9>(ad, rw, tg);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int r = w >> 1;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int y = tid + k * GCD_T;
                if (y < L[r]) W[w][y] = (live >> (2 * w + k)) & 1u ? uint32_t(rw[2 * w + k]) : 0u;
            }
        }
        if (c0 == s0) P[tid] = uint32_t(rw[8]);
        __syncthreads();

        const int items = 4 * (qn[0] + qn[1]);
        // selects instead of runtime-indexed arrays (those live in local memory)
        const int h00 = m.hi[0], h01 = m.hi[1], h10 = m.hi[2], h11 = m.hi[3];
        uint32_t* const W0 = W[0];
        uint32_t* const W1 = W[1];
        uint32_t* const W2 = W[2];
        uint32_t* const W3 = W[3];
        const int n0 = n[0], n1 = n[1], qn0 = qn[0];
        const long long xs0 = xs[0], xs1 = xs[1];
        uint64_t* const out0 = out[0];
        uint64_t* const out1 = out[1];
        for (int it0 = 0; it0 < items; it0 += GCD_T) {
            const int item = it0 + tid, q = item >> 2, part = item & 3;
            const int r = q < qn0 ? 0 : 1, qi = q - (r ? qn0 : 0);
            const int t = part >> 1, e0 = (part & 1) * (PL / 2);
            uint64_t acc[4] = {0, 0, 0, 0};
            uint32_t since = 0;
            const int h = r ? (t ? h11 : h10) : (t ? h01 : h00);
            if (item < items && h >= e0) {
                const int nblk = (min(h + 1, e0 + PL / 2) - e0 + 3) >> 2;
                uint32_t* const Wrt = r ? (t ? W3 : W2) : (t ? W1 : W0);
                conv_accumulate4_fast(acc, P + (2 * r + t) * PL + e0, nblk, Wrt,
                                   4 * qi + PL - 1 - e0, since, F);
            }
            uint32_t v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = reduce(acc[k], F);
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = addmod(v[k], __shfl_xor_sync(0xffffffffu, v[k], 1), F);
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = addmod(v[k], __shfl_xor_sync(0xffffffffu, v[k], 2), F);
            const int i = 4 * qi + part;  // part k stores output k of the quad
            if (item < items && i < (r ? n1 : n0)) {
                const uint32_t o = part == 0 ? v[0] : part == 1 ? v[1] : part == 2 ? v[2] : v[3];
                st_tag((r ? out1 + xs1 : out0 + xs0) + i, o, tg + 1u);
            }
        }
    }
}

// CTAs 1..G-1: apply batch j's matrix to this CTA's slice of both operands,
// S_{j+1} = P_j(S_j), as soon as its record is published (every record word
// polled until tagged j + 1: the matrix lands in shared memory, the meta in
// ms).  S_j's words are polled the same way inside apply_batch.
__device__ int bulk_cta(const GcdArgs& g, uint32_t* sm, int nbulk, int me) {
    __shared__ BatchMeta ms;
    long long apply_cycles = 0;  // MMM_GCD_STATS (bulk CTA 0, thread 0)
    long long ph[3] = {0, 0, 0}, seen_ns = 0, tseen0 = 0, warp_seen_ns = 0, nspin = 0, spin_ns = 0,
              tsw = 0, done_ns = 0;
    static_assert(REC_W <= 2 * GCD_T, "record: at most two words per thread");
    for (int j = 0;; ++j) {
        const uint64_t* rec = g.rec + (j % RING) * REC_W;
        const unsigned tg = unsigned(j + 1);
        // state buffer (j+1) % NBUF is free once every bulk CTA finished batch
        // j + 1 - NBUF (the head read S_{j+1-NBUF} before publishing that batch)
        // (normally the head's minimum in the record says so already)
        const unsigned need = j + 2 - NBUF > 0 ? unsigned(j + 2 - NBUF) : 0u;
        // the meta words (one cache line), polled by warp 0 alone: 147 CTAs
        // polling the whole record would queue the head's stores behind them
        const long long tpoll = (g.stats && me == 0) ? gtimer() : 0;
        if (threadIdx.x < 32) {
            const int l = threadIdx.x;
            const uint64_t* mp = rec + 4 * PL + (l < META_W ? l : 0);
            uint64_t w = ld_rlx64(mp);
            while (!__all_sync(0xffffffffu, unsigned(w >> 32) == tg)) {
                if (g.dbg & 2) __nanosleep(256);
                w = ld_rlx64(mp);
            }
            if (g.stats && me == 0 && l == 0) tseen0 = gtimer();
            static_assert(sizeof(BatchMeta) == META_W * sizeof(int), "meta words = BatchMeta");
            if (l < META_W) reinterpret_cast<int*>(&ms)[l] = int(uint32_t(w));
            __syncwarp();
            if (g.stats && me == 0 && l == 0) tsw = gtimer();
        }
        __syncthreads();  // the meta (the matrix words are read with S_j in apply_batch)
        long long tg0 = (g.stats && me == 0 && threadIdx.x == 0) ? gtimer() : 0;
        if (ms.minprog < need) {  // uniform; rare
            if (threadIdx.x < 32)
                while (min_progress(g.prog, nbulk) < need) {
                }
            __syncthreads();
            if (g.stats && me == 0) nspin += 1;
        }
        if (g.stats && me == 0 && threadIdx.x == 0) ph[2] += gtimer() - tg0;
        const long long mtp = (long long)(((unsigned long long)(unsigned)ms.tpub_hi << 32) |
                                          (unsigned)ms.tpub_lo);
        if (g.stats && me == 0 && threadIdx.x == 0) {
            const long long now = gtimer();
            seen_ns += now - mtp;
            warp_seen_ns += tseen0 - mtp;
            spin_ns += tsw - tseen0;
            ph[1] += now - (tpoll > mtp ? tpoll : mtp);  // poll latency once published
        }
        if (g.stats && me == nbulk - 1 && threadIdx.x == 0) seen_ns += gtimer() - mtp;
        const long long tb = clock64();
        const BatchMeta& m = ms;  // shared: runtime-indexed fields stay out of local memory
        if (m.steps > 0 && !m.err) {
            const long long na1 = m.da1 + 1 > 0 ? m.da1 + 1 : 0;
            const long long nb1 = m.db1 + 1 > 0 ? m.db1 + 1 : 0;
            const long long per = (na1 + nb1 + nbulk - 1) / nbulk;
            const long long s0 = min((long long)me * per, na1 + nb1);
            const long long s1 = min(s0 + per, na1 + nb1);
            apply_batch(g, m, j, s0, s1, sm, rec, (g.stats && me == 0 && threadIdx.x == 0) ? ph : nullptr);
        }
        const bool last = m.term || m.err;
        __syncthreads();  // sm and ms reused by the next batch
        if (threadIdx.x == 0) {
            // finished reading S_j and record j (the ring guards).  No release:
            // those reads are complete (their values were consumed before the
            // barrier above), and a fence costs ~1 us on this part.
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(g.prog + me), "r"(unsigned(j + 1))
                         : "memory");
            apply_cycles += clock64() - tb;
            if (g.stats && me == nbulk - 1) done_ns += gtimer() - mtp;
        }
        if (last) {
            if (g.stats && me == 0 && threadIdx.x == 0) {
                g.stats[7] = apply_cycles;
                g.stats[12] = seen_ns;
                g.stats[16] = nspin;
                g.stats[14] = spin_ns;
                g.stats[13] = warp_seen_ns;
                g.stats[14] = spin_ns;
                g.stats[15] = ph[2];
            }
            if (g.stats && me == nbulk - 1 && threadIdx.x == 0) {
                g.stats[18] = seen_ns;
                g.stats[20] = done_ns;
            }
            return j;
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(GCD_T, 1) gcd_kernel(GcdArgs g) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ BatchMeta ctl, fin;
    __shared__ int hi_s[4];
    __shared__ volatile int done;
    cg::grid_group grid = cg::this_grid();
    const FieldParams F = g.F;
    const long long tid = (long long)blockIdx.x * GCD_T + threadIdx.x;
    const long long nth = (long long)gridDim.x * GCD_T;
    const int nbulk = gridDim.x - 1;  // >= 1 (launcher)
    StepLog* log = reinterpret_cast<StepLog*>(smem);
    uint32_t* rest = smem + 4 * LOGCAP;

    // S_0 tagged 1; every other state word and record word untagged (0), so
    // no tag left by an earlier call can be mistaken for this one's
    for (long long i = tid; i < g.cap; i += nth) {
        g.XA[0][i] = i < g.na ? (uint64_t(1) << 32) | g.a[i] : 0ull;
        g.XB[0][i] = i < g.nb ? (uint64_t(1) << 32) | g.b[i] : 0ull;
#pragma unroll
        for (int r = 1; r < NBUF; ++r) g.XA[r][i] = g.XB[r][i] = 0ull;
    }
    for (long long i = tid; i < RING * REC_W; i += nth) g.rec[i] = 0ull;
    grid.sync();

    const int J = blockIdx.x == 0 ? head_cta<MODE>(g, ctl, log, rest, &done, hi_s, nbulk)
                                  : bulk_cta(g, rest, nbulk, blockIdx.x - 1);
    // every CTA: the final record, then the final state (tagged reads wait for it)
    if (threadIdx.x < 8) {
        const int v = int(ld_tag(g.rec + (J % RING) * REC_W + 4 * PL + threadIdx.x, unsigned(J + 1)));
        if (threadIdx.x == 2) fin.da1 = v;
        if (threadIdx.x == 3) fin.db1 = v;
        if (threadIdx.x == 4) fin.steps = v;
        if (threadIdx.x == 5) fin.term = v;
        if (threadIdx.x == 7) fin.err = v;
    }
    __syncthreads();
    if (fin.err) {
        if (tid == 0) *g.ng = -2;  // no progress: internal invariant broken
        return;
    }
    if (fin.term == 3) {
        if (tid == 0) {
            g.g[0] = 1u;
            *g.ng = 1;
        }
        return;
    }
    const int buf = fin.steps > 0 ? (J + 1) % NBUF : J % NBUF;
    const unsigned tg = fin.steps > 0 ? unsigned(J + 2) : unsigned(J + 1);
    const uint64_t* Z = fin.term == 1 ? g.XB[buf] : g.XA[buf];
    const long long dz = fin.term == 1 ? fin.db1 : fin.da1;
    const uint32_t inv = invmod(ld_tag(Z + dz, tg), F);
    for (long long i = tid; i <= dz; i += nth) g.g[i] = mulmod(ld_tag(Z + i, tg), inv, F);
    if (tid == 0) *g.ng = dz + 1;
}

void launch_gcd(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb,
                uint32_t* gout, int64_t* d_ng, int64_t s, cudaStream_t st) {
    if (s < 1) throw Error(ST_INVALID, "gcd: s must be >= 1");
    GcdArgs g{};
    g.a = a;
    g.b = b;
    g.na = na;
    g.nb = nb;
    g.g = gout;
    g.ng = d_ng;
    g.F = F;
    g.M = int(std::min<int64_t>(s, LOGCAP));
    const int64_t cap = std::max<int64_t>(std::max(na, nb), 1);
    Scratch sc(st);
    for (int i = 0; i < NBUF; ++i) {
        g.XA[i] = sc.get<uint64_t>(size_t(cap));
        g.XB[i] = sc.get<uint64_t>(size_t(cap));
    }
    g.cap = cap;
    g.rec = sc.get<uint64_t>(size_t(RING) * REC_W);
    g.prog = sc.get<unsigned>(MAXBULK);
    MMM_CUDA(cudaMemsetAsync(g.prog, 0, MAXBULK * sizeof(unsigned), st));
    const size_t head_words = 2 * W1 + 2 * (W1 + PL) + 4 * PL + BUILD_PARTS * 2 * W1;
    const size_t bulk_words = APPLY_WORDS;
    const size_t bytes = (4 * LOGCAP + std::max(head_words, bulk_words)) * 4;
    const int mode = !F.odd ? 2 : (F.p < (1u << 29) ? 0 : 1);
    const void* fn = mode == 0 ? (const void*)gcd_kernel<0>
                               : (mode == 1 ? (const void*)gcd_kernel<1> : (const void*)gcd_kernel<2>);
    // attribute and occupancy once per (device, flavour): host time in every e2e call otherwise
    static std::mutex fit_mu;
    static std::map<std::pair<int, int>, int> fit;
    int dev = 0;
    MMM_CUDA(cudaGetDevice(&dev));
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lock(fit_mu);
        auto it = fit.find({dev, mode});
        if (it == fit.end()) {
            MMM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
            MMM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, GCD_T, bytes));
            fit[{dev, mode}] = per_sm;
        } else {
            per_sm = it->second;
        }
    }
    if (per_sm < 1) throw Error(ST_INVALID, "gcd: kernel does not fit an SM");
    const int64_t want = std::max<int64_t>(2, 1 + ceil_div(na + nb, GCD_OUT_PER_CTA));
    // one CTA per SM: a second CTA on the head's SM would take issue slots from the chain
    const int blocks = int(std::min<int64_t>(std::min<int64_t>(want, int64_t(sm_count())), MAXBULK + 1));
    const bool want_stats = getenv("MMM_GCD_STATS") != nullptr;
    if (const char* d = getenv("MMM_GCD_DEBUG")) g.dbg = atoi(d);
    if (want_stats) {
        g.stats = sc.get<long long>(32);
        MMM_CUDA(cudaMemsetAsync(g.stats, 0, 32 * sizeof(long long), st));
    }
    void* params[] = {&g};
    MMM_CUDA(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(GCD_T), params, bytes, st));
    check_launch("gcd_kernel", dim3(blocks), dim3(GCD_T));
    if (want_stats) {
        long long h[32];
        MMM_CUDA(cudaMemcpyAsync(h, g.stats, sizeof(h), cudaMemcpyDeviceToHost, st));
        MMM_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr,
                "gcd stats: blocks=%d batches=%lld steps=%lld phase_end_cycles=%lld "
                "head_total_cycles=%lld chain_warp_cycles=%lld replay_warp_cycles=%lld "
                "prefetch_cycles=%lld bulk0_apply_cycles=%lld builder_own_done=%lld "
                "builders_synced=%lld\n",
                blocks, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9]);
        fprintf(stderr,
                "gcd latency: bulk0_seen_ns=%lld bulk0_warp_seen_ns=%lld bulk0_switch_ns=%lld "
                "bulk0_barrier_ns=%lld spins=%lld head_prefetch_seen_ns=%lld (%lld) bulkLast_seen_ns=%lld replay_loop_exit_cyc=%lld bulkLast_done_ns=%lld build_start=%lld build_part_done=%lld windows_ready=%lld warm_rebuild=%lld\n",
                h[12], h[13], h[14], h[15], h[16], h[17], h[19], h[18], h[10], h[20], h[21], h[22], h[23], h[24]);
    }
}

}  // namespace mmm_cu
