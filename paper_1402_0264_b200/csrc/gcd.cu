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
#include <cstdlib>

namespace cg = cooperative_groups;

namespace mmm_cu {

constexpr int GCD_T = 256;         // threads per CTA
constexpr int GE = 4;              // window words per lane
constexpr int W1 = 32 * GE;        // window words per operand (128)
constexpr int PE = 4;              // matrix words per lane per polynomial
constexpr int PL = 32 * PE;        // matrix capacity (support < 128)
constexpr int LOGCAP = 2048;       // steps per matrix batch, hard cap
constexpr int BIG = 1 << 30;       // "validity unbounded": window covers the operand
constexpr int GCD_R = 1;           // outputs per thread in the apply

struct StepLog {
    uint32_t x, y;
    int z;       // renormalisation shift of the reduced operand
    int u_is_a;  // 1: A was reduced by B, 0: B by A
};

// Published per batch by CTA 0 (global), read by every CTA after the barrier.
struct BatchMeta {
    long long da0, db0;  // exact degrees at batch start (-1: zero operand)
    long long da1, db1;  // degree bounds after the batch (-1: vanished)
    int steps, term, dividend_a, err;
    int sa, sb;          // total shifts of A and B (top moves)
    int hi[4];           // highest nonzero index of Pa1, Pa2, Pb1, Pb2
};

struct GcdArgs {
    const uint32_t* a;
    const uint32_t* b;
    long long na, nb;
    uint32_t* X[2];
    uint32_t* Y[2];
    uint32_t* Pg;     // 4 * PL words: Pa1, Pa2, Pb1, Pb2 (canonical)
    BatchMeta* meta;  // global copy
    uint32_t* g;
    int64_t* ng;
    int M;            // steps per batch (the program parameter s)
    FieldParams F;
    long long* stats; // optional (MMM_GCD_STATS): batches, steps, chain/apply cycles
    int dbg;          // MMM_GCD_DEBUG bits (timing experiments; 2 = serialise chain and replay)
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

// Load the top W1 words of Z below `deg` into w; lower `deg` past zero words
// until w[0] is the nonzero lead (or deg = -1: zero operand).  Warp-uniform.
template <int MODE>
__device__ void load_top(uint32_t (&w)[GE], const uint32_t* Z, long long& deg, uint32_t p) {
    const int lane = threadIdx.x & 31;
    while (deg >= 0) {
#pragma unroll
        for (int e = 0; e < GE; ++e) {
            const long long x = deg - (e * 32 + lane);
            w[e] = x >= 0 ? __ldcg(Z + x) : 0u;
        }
        const int z = first_nz<MODE>(w, 0, p);
        if (z == 0) return;
        deg -= z < 0 ? W1 : z;
    }
}

// Log entries: the chain buffers entry s in lane s % 32 and stores 32 at a
// time, one 16-byte store per lane; `seq` = step index + 1 publishes an entry
// (the replay warps poll the entry itself, no per-step fence or store).
__device__ __forceinline__ void log_flush(StepLog* log, int base, int count, uint32_t x,
                                          uint32_t y, uint32_t zf) {
    const int lane = threadIdx.x & 31;
    if (lane < count) {
        const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(log + base + lane));
        asm volatile("st.volatile.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y),
                     "r"(zf), "r"(unsigned(base + lane + 1))
                     : "memory");
    }
}
__device__ __forceinline__ uint4 log_get(const StepLog* log, int i) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(const_cast<StepLog*>(log + i)));
    uint4 v;
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a)
                 : "memory");
    return v;
}

// Warp 0 of CTA 0: the elimination chain of one batch.  Windows are kept
// oriented: u = current dividend, v = divisor (roles swap with MOVs only, so
// every shuffle sits in straight-line, warp-uniform code).  Fast path: the
// new lead is u[1] (z = 1), fetched by one shuffle while the window shifts
// by one; all capacity checks collapse into one budget counter F of steps
// that provably cannot exhaust the windows or the matrix.
template <int MODE>
__device__ void run_chain(BatchMeta& c, StepLog* log, volatile int* done, int M, Fld f,
                          const uint32_t* X, const uint32_t* Y) {
    using A = Arith<MODE>;
    const uint32_t p = f.p;
    long long da = c.da1, db = c.db1;
    uint32_t u[GE], v[GE];
    load_top<MODE>(u, X, da, p);
    load_top<MODE>(v, Y, db, p);
    const long long da0 = da, db0 = db;
    bool u_is_a = true;
    int du = int(da), dv = int(db);
    int vu = da < W1 ? BIG : W1, vv = db < W1 ? BIG : W1;
    int su = 0, sv = 0, supu = 0, supv = 0;
    uint32_t hu = bcast(u[0]), hv = bcast(v[0]);
    auto swap_roles = [&]() {
#pragma unroll
        for (int e = 0; e < GE; ++e) {
            const uint32_t t = u[e];
            u[e] = v[e];
            v[e] = t;
        }
        u_is_a = !u_is_a;
        int t;
        t = du; du = dv; dv = t;
        t = vu; vu = vv; vv = t;
        t = su; su = sv; sv = t;
        t = supu; supu = supv; supv = t;
        const uint32_t h = hu; hu = hv; hv = h;
    };
    if (!c.dividend_a) swap_roles();
    const int cap = min(M, LOGCAP);
    const int lane = threadIdx.x & 31;
    int steps = 0, term = 0, F = 0;
    uint32_t lx = 0, ly = 0, lz = 0;  // this lane's buffered log entry
    for (;;) {
        if (du >= 0 && dv >= 0 && du < dv) swap_roles();  // oracle.cpp:58-66, 74-75
        if (F <= 0) {
            if (du < 0) { term = u_is_a ? 1 : 2; break; }  // dividend vanished: gcd = divisor
            if (dv < 0) { term = u_is_a ? 2 : 1; break; }  // zero divisor (zero input)
            F = min(cap - steps, min(min(vu, vv) - 2, PL - 2 - max(supu, supv)));
            if (F <= 0) break;  // batch length, window or matrix exhausted
        }
        if (dv == 0) { term = 3; break; }  // constant divisor: unit gcd
        const uint32_t x = hu, y = hv, nx = A::neg(x, p);
        vu = min(vu, vv);
#pragma unroll
        for (int e = 0; e < GE; ++e) u[e] = A::comb(y, u[e], nx, v[e], f);
        const uint32_t h1 = from_lane(u[0], 1);
        int z = 1;
        bool stop = false;
        if (A::nz(h1, p)) {  // fast path: the next word is the new lead
            shift_left1(u, GE);
            hu = h1;
            --F;
        } else {
            z = first_nz<MODE>(u, 1, p);
            if (z < 0 || z >= vu) {
                if (vu >= BIG) {  // window held the whole operand: it vanished
                    du = -1;
                    z = 0;
                } else {          // lead not determined inside the valid words
                    z = vu;
                    stop = true;
                }
            }
            const int room = PL - 1 - max(supu, supv);
            if (z > room) {       // matrix capacity: shift only as far as it holds
                z = room;
                stop = true;
            }
            if (du >= 0) {
                shift_left(u, z);
                hu = bcast(u[0]);
            }
            F = 0;                // re-derive the budget
        }
        if (du >= 0) {
            du -= z;
            if (vu < BIG) vu -= z;
        }
        su += z;
        supu = max(supu, supv) + z;
        // buffer the log entry in lane (steps % 32); flush 32 at a time
        if (lane == (steps & 31)) {
            lx = x;
            ly = y;
            lz = unsigned(z) | (u_is_a ? 0x10000u : 0u);
        }
        ++steps;
        if ((steps & 31) == 0) log_flush(log, steps - 32, 32, lx, ly, lz);
        if (stop) break;
    }
    if (steps & 31) log_flush(log, steps & ~31, steps & 31, lx, ly, lz);
    if ((threadIdx.x & 31) == 0) {
        c.da0 = da0;
        c.db0 = db0;
        c.da1 = u_is_a ? du : dv;
        c.db1 = u_is_a ? dv : du;
        c.steps = steps;
        c.term = term;
        c.dividend_a = u_is_a ? 1 : 0;
        c.sa = u_is_a ? su : sv;
        c.sb = u_is_a ? sv : su;
        st_release_cta(done, steps + 1);  // done = final count + 1
    }
}

// Warps 1 and 2 of CTA 0: replay the step log into matrix column `col`
// (both rows), oriented like the chain; then publish it (canonical) to Pg.
template <int MODE>
__device__ void run_replay(int col, const StepLog* log, volatile int* done, Fld f, uint32_t* Pg,
                           int* hi_out) {
    using A = Arith<MODE>;
    const uint32_t p = f.p;
    const int lane = threadIdx.x & 31;
    uint32_t ru[PE], rv[PE];  // rows of the operands held in the chain's u / v
#pragma unroll
    for (int e = 0; e < PE; ++e) ru[e] = rv[e] = 0u;
    if (lane == 0) {  // identity: row A col 0 = 1, row B col 1 = 1; oriented u = A
        if (col == 0) ru[0] = 1u;
        else rv[0] = 1u;
    }
    bool u_is_a = true;
    int hu = col == 0 ? 0 : -1, hv = col == 0 ? -1 : 0;
    for (int i = 0;; ++i) {
        uint4 en = log_get(log, i);
        while (en.w != unsigned(i + 1)) {
            const int d = ld_acquire_cta(done);
            if (d != 0 && d - 1 <= i) break;  // chain finished with i entries
            __nanosleep(32);
            en = log_get(log, i);
        }
        if (en.w != unsigned(i + 1)) break;
        const bool sa = (en.z >> 16) != 0;
        const int z = int(en.z & 0xFFFFu);
        if (sa != u_is_a) {
#pragma unroll
            for (int e = 0; e < PE; ++e) {
                const uint32_t t = ru[e];
                ru[e] = rv[e];
                rv[e] = t;
            }
            const int t = hu; hu = hv; hv = t;
            u_is_a = sa;
        }
        const uint32_t nx = A::neg(en.x, p);
        const int hmax = max(hu, hv);
#pragma unroll
        for (int e = 0; e < PE; ++e) ru[e] = A::comb(en.y, ru[e], nx, rv[e], f);
        if (z == 1) shift_right1(ru, PE);
        else shift_right(ru, z);
        hu = hmax;
        if (hu >= 0) hu += z;
    }
    uint32_t* Pa = Pg + (0 * 2 + col) * PL;  // row A, column col
    uint32_t* Pb = Pg + (1 * 2 + col) * PL;  // row B, column col
#pragma unroll
    for (int e = 0; e < PE; ++e) {
        __stcg(Pa + e * 32 + lane, A::canon(u_is_a ? ru[e] : rv[e], p));
        __stcg(Pb + e * 32 + lane, A::canon(u_is_a ? rv[e] : ru[e], p));
    }
    if (lane == 0) {
        hi_out[0 * 2 + col] = min(u_is_a ? hu : hv, PL - 1);
        hi_out[1 * 2 + col] = min(u_is_a ? hv : hu, PL - 1);
    }
}

// out[x] = sum_{e<=h1} P1[e] Z1[x + s1 - e] + sum_{e<=h2} P2[e] Z2[x + s2 - e],
// x in [xs, xe); Zi[j] = 0 outside [0, bi].  One CTA, all threads.
__device__ void apply_row(uint32_t* out, long long xs, long long xe, const uint32_t* P1, int h1,
                          const uint32_t* Z1, long long b1, long long s1, const uint32_t* P2,
                          int h2, const uint32_t* Z2, long long b2, long long s2, uint32_t* sw,
                          uint32_t* sv, int ORG, const FieldParams& F) {
    constexpr int R = GCD_R;
    const long long n = xe - xs;
    if (n <= 0) return;
    for (long long c0 = 0; c0 < n; c0 += (long long)GCD_T * R) {
        const long long cn = min(n - c0, (long long)GCD_T * R);
        uint64_t acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0;
        uint32_t since = 0;
        for (int term = 0; term < 2; ++term) {
            const int h = term ? h2 : h1;
            if (h < 0) continue;
            const uint32_t* Pt = term ? P2 : P1;
            const uint32_t* Zt = term ? Z2 : Z1;
            const long long zb = term ? b2 : b1;
            const long long off = xs + c0 + (term ? s2 : s1) - ORG;  // sv[y] = Zt[y + off]
            const int width = h + 1, wpad = (width + R - 1) / R * R;
            __syncthreads();
            for (int u = threadIdx.x; u < wpad; u += GCD_T) sw[u] = u < width ? __ldcg(Pt + u) : 0u;
            for (long long y = threadIdx.x; y < ORG + cn + R; y += GCD_T) {
                const long long x = y + off;
                sv[y] = (x >= 0 && x <= zb) ? __ldcg(Zt + x) : 0u;
            }
            __syncthreads();
            const long long y0 = (long long)threadIdx.x * R;
            if (y0 < cn) conv_accumulate<R>(acc, sw, wpad / R, sv, int(ORG + y0), since, F);
        }
        const long long y0 = (long long)threadIdx.x * R;
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (y0 + r < cn) __stcg(out + xs + c0 + y0 + r, reduce(acc[r], F));
    }
}

}  // namespace

template <int MODE>
__global__ void __launch_bounds__(GCD_T, 1) gcd_kernel(GcdArgs g) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ BatchMeta ctl;
    __shared__ int hi_s[4];
    __shared__ volatile int done;
    cg::grid_group grid = cg::this_grid();
    const FieldParams F = g.F;
    constexpr int ORG = PL + 8 + 3;
    StepLog* log = reinterpret_cast<StepLog*>(smem);                 // LOGCAP entries
    uint32_t* sw = smem + 4 * LOGCAP;                                 // PL + 8 words
    uint32_t* sv = sw + PL + 8;                                       // ORG + GCD_T*R + R
    const long long tid = (long long)blockIdx.x * GCD_T + threadIdx.x;
    const long long nth = (long long)gridDim.x * GCD_T;
    const int warp = threadIdx.x >> 5;

    for (long long i = tid; i < g.na; i += nth) g.X[0][i] = g.a[i];
    for (long long i = tid; i < g.nb; i += nth) g.Y[0][i] = g.b[i];
    if (threadIdx.x == 0) {
        ctl.da1 = g.na - 1;
        ctl.db1 = g.nb - 1;
        ctl.dividend_a = 1;  // oracle_gcd: x = a is the first dividend (oracle.cpp:70)
    }
    grid.sync();

    int cur = 0;
    for (;;) {
        long long t_chain0 = clock64();
        if (blockIdx.x == 0) {
            for (int i = threadIdx.x; i < LOGCAP; i += GCD_T)
                reinterpret_cast<uint4*>(log)[i] = make_uint4(0u, 0u, 0u, 0u);
            if (threadIdx.x == 0) done = 0;
            __syncthreads();
            if (warp == 0) {
                run_chain<MODE>(ctl, log, &done, g.M, Fld{F.p, F.pinv},
                                (cur ? g.X[1] : g.X[0]), (cur ? g.Y[1] : g.Y[0]));
                if (g.stats && threadIdx.x == 0) g.stats[4] += clock64() - t_chain0;
            }
            else if (warp <= 2) {
                if (g.dbg & 2)  // experiment: replay only after the chain finished
                    while (ld_acquire_cta(&done) == 0) __nanosleep(256);
                run_replay<MODE>(warp - 1, log, &done, Fld{F.p, F.pinv}, g.Pg, hi_s);
                if (g.stats && threadIdx.x == 32) g.stats[5] += clock64() - t_chain0;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                BatchMeta m = ctl;
                for (int i = 0; i < 4; ++i) m.hi[i] = hi_s[i];
                m.err = 0;
                *g.meta = m;
                __threadfence();
                if (g.stats) {
                    g.stats[0] += 1;
                    g.stats[1] += ctl.steps;
                    g.stats[2] += clock64() - t_chain0;
                }
            }
        }
        grid.sync();
        // one reader per CTA: every thread polling the same global line would
        // serialise ~25k requests on one L2 slice per batch
        __shared__ BatchMeta ms;
        if (threadIdx.x == 0) {
            const volatile BatchMeta* vm = g.meta;
            ms.da0 = vm->da0; ms.db0 = vm->db0; ms.da1 = vm->da1; ms.db1 = vm->db1;
            ms.steps = vm->steps; ms.term = vm->term; ms.dividend_a = vm->dividend_a;
            ms.sa = vm->sa; ms.sb = vm->sb;
            for (int i = 0; i < 4; ++i) ms.hi[i] = vm->hi[i];
        }
        __syncthreads();
        const BatchMeta m = ms;
        if (m.steps == 0 && m.term == 0) {  // invariant broken: no progress
            if (tid == 0) *g.ng = -2;
            return;                         // grid-uniform
        }
        if (m.term == 3) break;
        if (m.steps > 0) {
            const long long na1 = m.da1 + 1 > 0 ? m.da1 + 1 : 0;
            const long long nb1 = m.db1 + 1 > 0 ? m.db1 + 1 : 0;
            const long long per = (na1 + nb1 + gridDim.x - 1) / gridDim.x;
            const long long s0 = (long long)blockIdx.x * per;
            const long long s1 = min(s0 + per, na1 + nb1);
            // A1[x] = Pa1 * A0 (shift sa) + Pa2 * B0 (shift sa + db0 - da0)
            apply_row((cur ? g.X[0] : g.X[1]), min(s0, na1), min(s1, na1), g.Pg + 0 * PL, m.hi[0],
                      (cur ? g.X[1] : g.X[0]), m.da0, m.sa, g.Pg + 1 * PL, m.hi[1], (cur ? g.Y[1] : g.Y[0]), m.db0,
                      m.sa + m.db0 - m.da0, sw, sv, ORG, F);
            // B1[x] = Pb1 * A0 (shift sb + da0 - db0) + Pb2 * B0 (shift sb)
            apply_row((cur ? g.Y[0] : g.Y[1]), max(s0 - na1, 0LL), max(s1 - na1, 0LL), g.Pg + 2 * PL,
                      m.hi[2], (cur ? g.X[1] : g.X[0]), m.da0, m.sb + m.da0 - m.db0, g.Pg + 3 * PL, m.hi[3],
                      (cur ? g.Y[1] : g.Y[0]), m.db0, m.sb, sw, sv, ORG, F);
            grid.sync();
            if (g.stats && tid == 0) g.stats[3] += clock64() - t_chain0;
            cur ^= 1;
        }
        if (m.term) {
            ctl.term = m.term;
            ctl.da1 = m.da1;
            ctl.db1 = m.db1;
            break;
        }
    }
    __syncthreads();
    __shared__ BatchMeta fs;
    if (threadIdx.x == 0) {
        const volatile BatchMeta* vm = g.meta;
        fs.term = vm->term;
        fs.da1 = vm->da1;
        fs.db1 = vm->db1;
    }
    __syncthreads();
    const BatchMeta fin = fs;
    if (fin.term == 3) {
        if (tid == 0) {
            g.g[0] = 1u;
            *g.ng = 1;
        }
        return;
    }
    const uint32_t* Z = fin.term == 1 ? (cur ? g.Y[1] : g.Y[0]) : (cur ? g.X[1] : g.X[0]);
    const long long dz = fin.term == 1 ? fin.db1 : fin.da1;
    const uint32_t inv = invmod(__ldcg(Z + dz), F);
    for (long long i = tid; i <= dz; i += nth) g.g[i] = mulmod(__ldcg(Z + i), inv, F);
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
    for (int i = 0; i < 2; ++i) {
        g.X[i] = sc.get<uint32_t>(size_t(cap));
        g.Y[i] = sc.get<uint32_t>(size_t(cap));
    }
    g.Pg = sc.get<uint32_t>(4 * PL);
    g.meta = reinterpret_cast<BatchMeta*>(sc.get<uint64_t>((sizeof(BatchMeta) + 7) / 8));
    constexpr int ORG = PL + 8 + 3;
    const size_t bytes = size_t(4 * LOGCAP + PL + 8 + ORG + GCD_T * GCD_R + GCD_R + 8) * 4;
    const int mode = !F.odd ? 2 : (F.p < (1u << 29) ? 0 : 1);
    const void* fn = mode == 0 ? (const void*)gcd_kernel<0>
                               : (mode == 1 ? (const void*)gcd_kernel<1> : (const void*)gcd_kernel<2>);
    MMM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    int per_sm = 0;
    MMM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, GCD_T, bytes));
    if (per_sm < 1) throw Error(ST_INVALID, "gcd: kernel does not fit an SM");
    const int64_t want = std::max<int64_t>(1, ceil_div(na + nb, 256));
    const int blocks = int(std::min<int64_t>(want, int64_t(sm_count()) * per_sm));
    const bool want_stats = getenv("MMM_GCD_STATS") != nullptr;
    if (const char* d = getenv("MMM_GCD_DEBUG")) g.dbg = atoi(d);
    if (want_stats) {
        g.stats = sc.get<long long>(6);
        MMM_CUDA(cudaMemsetAsync(g.stats, 0, 6 * sizeof(long long), st));
    }
    void* params[] = {&g};
    MMM_CUDA(cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(GCD_T), params, bytes, st));
    check_launch("gcd_kernel");
    if (want_stats) {
        long long h[6];
        MMM_CUDA(cudaMemcpyAsync(h, g.stats, sizeof(h), cudaMemcpyDeviceToHost, st));
        MMM_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr,
                "gcd stats: blocks=%d batches=%lld steps=%lld cta0_cycles=%lld total_cycles=%lld "
                "chain_warp_cycles=%lld replay_warp_cycles=%lld\n",
                blocks, h[0], h[1], h[2], h[3], h[4], h[5]);
    }
}

}  // namespace mmm_cu
