// gcd.cu -- Euclidean GCD over Z/pZ on sm_100a, s elimination steps per batch.
//
// Result: exactly oracle_gcd (proj/src/oracle.cpp:69-78), the monic gcd.
// Structure: the paper's optimized GCD (Alg. 9-10) as simulated by
// run_gcd's optimized variant (proj/src/gcd.cpp:116-330): up to s head
// eliminations are folded into a 2x2 matrix of offset polynomials
// (UpdateMatrix, gcd.cpp:124-157) that is then applied to both operands by
// every block.  Differences, B200-first:
//
//  * The matrix is staged ON DEVICE (the reference stages it on the host,
//    reading device memory per launch, gcd.cpp:203-272).  Warp 0 of every CTA
//    runs the step chain redundantly on the operands' top windows in shared
//    memory -- the paper's redundant s-head computation -- so there is no
//    host round trip and no extra grid barrier to broadcast the matrix.
//  * Steps are fraction-free:  A <- y*A - x*X^k*B  (x, y the two leads),
//    evaluated as one Montgomery reduction of y*a + (p-x)*b, i.e. up to the
//    unit 2^-32.  No per-step field inverse; the operands stay associates of
//    the oracle's remainders, so the final monic result is bit-identical.
//  * The role rule is the oracle's: the dividend keeps being reduced while
//    deg(dividend) >= deg(divisor) (divmod's i-loop, oracle.cpp:58-66), then
//    the roles swap (oracle.cpp:74-75); a zero dividend ends the run with the
//    divisor as gcd, a degree-0 divisor with gcd 1 (gcd.cpp:191-199).
//  * One persistent cooperative grid; a batch = chain, matrix apply
//    (conv.cuh convolutions over L2-resident ping-pong buffers), grid barrier.
//
// Offset convention (as OffPoly): wa[j] = A[da0 - j], wb[j] = B[db0 - j] for
// the batch-start degree bounds da0, db0.  New operands are
//   A1[da0-j] = sum_d P11[d] wa0[j-d] + sum_d P12[d] wb0[j-d]   (same for B)
// with every P support inside [-W, W].
#include <cooperative_groups.h>

#include "common.cuh"
#include "conv.cuh"

namespace cg = cooperative_groups;

namespace mmm_cu {

constexpr int GCD_T = 256;
constexpr int GCD_R = 2;

struct GcdArgs {
    const uint32_t* a;
    const uint32_t* b;
    int64_t na, nb;
    uint32_t* X[2];
    uint32_t* Y[2];
    uint32_t* g;
    int64_t* ng;
    int64_t cap;  // words per buffer
    int S;        // steps per batch
    int W;        // window words per operand
    FieldParams F;
};

// Shared-memory control block written by warp 0, read by the whole CTA.
struct GcdCtl {
    int64_t da0, db0;   // batch-start degree bounds (offset origins)
    int64_t da1, db1;   // bounds after the batch (-1: operand vanished)
    int lo[4], hi[4];   // P supports (d), lo > hi = empty
    int steps;
    int term;           // 0 running, 1 A vanished, 2 B vanished, 3 unit gcd
    int dividend_a;
    int err;
};

namespace {

__device__ __forceinline__ int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t i64max(int64_t a, int64_t b) { return a > b ? a : b; }

// Warp-wide: first j in [from, to) with w[j] != 0, else -1.
__device__ int first_nonzero(const uint32_t* w, int from, int to) {
    const int lane = threadIdx.x & 31;
    for (int base = from; base < to; base += 32) {
        const int j = base + lane;
        const unsigned m = __ballot_sync(0xffffffffu, j < to && w[j] != 0);
        if (m) return base + __ffs(m) - 1;
    }
    return -1;
}

// Load the top W words below `bound` of buffer Z into w (zero below index 0),
// lowering the bound past all-zero windows.  Returns the head offset, or -1
// if the operand is zero.  `bound` is updated (warp-uniform).
__device__ int load_window(uint32_t* w, const uint32_t* Z, int64_t& bound, int W) {
    const int lane = threadIdx.x & 31;
    while (bound >= 0) {
        for (int j = lane; j < W; j += 32) {
            const int64_t x = bound - j;
            w[j] = x >= 0 ? __ldcg(Z + x) : 0u;
        }
        __syncwarp();
        const int u = first_nonzero(w, 0, W);
        if (u >= 0) return u;
        bound -= W;
        __syncwarp();
    }
    return -1;
}

// dst[d] <- y*dst[d] - x*src[d - delta]  over the union support (fraction-free).
__device__ void p_update(uint32_t* dst, int& dlo, int& dhi, const uint32_t* src, int slo, int shi,
                         int delta, uint32_t y, uint32_t negx, int W, const FieldParams& F,
                         int& err) {
    const int lane = threadIdx.x & 31;
    int lo = dlo, hi = dhi;
    if (slo <= shi) {
        lo = min(lo, slo + delta);
        hi = max(hi, shi + delta);
    }
    if (lo < -W || hi > W) {
        err = 1;
        return;
    }
    for (int d = lo + lane; d <= hi; d += 32) {
        const int e = d - delta;
        const uint32_t sv = (e >= slo && e <= shi) ? src[e + W] : 0u;
        const uint32_t dv = (d >= dlo && d <= dhi) ? dst[d + W] : 0u;
        dst[d + W] = ff_comb(y, dv, negx, sv, F);
    }
    dlo = lo;
    dhi = hi;
    __syncwarp();
}

// The step chain of one batch, run by warp 0 (all lanes active).
__device__ void run_chain(GcdCtl& c, uint32_t* wa, uint32_t* wb, uint32_t* P, const GcdArgs& g,
                          const uint32_t* X, const uint32_t* Y) {
    const int W = g.W;
    const int PL = 2 * W + 1;
    const FieldParams F = g.F;
    const int lane = threadIdx.x & 31;
    int64_t da0 = c.da1, db0 = c.db1;
    int ua = load_window(wa, X, da0, W);
    int ub = load_window(wb, Y, db0, W);
    for (int i = lane; i < 4 * PL; i += 32) P[i] = 0u;
    __syncwarp();
    if (lane == 0) {
        P[0 * PL + W] = 1u;  // P11 = 1
        P[3 * PL + W] = 1u;  // P22 = 1
    }
    __syncwarp();
    int lo[4] = {0, 1, 1, 0}, hi[4] = {0, 0, 0, 0};
    int limA = W, limB = W, steps = 0, term = 0, err = 0;
    int dividend_a = c.dividend_a;
    int64_t da = ua < 0 ? -1 : da0 - ua;
    int64_t db = ub < 0 ? -1 : db0 - ub;
    bool unknown = false;
    while (steps < g.S && !unknown) {
        if (da < 0) { term = 1; break; }
        if (db < 0) { term = 2; break; }
        if (dividend_a && da < db) dividend_a = 0;
        else if (!dividend_a && db < da) dividend_a = 1;
        if ((dividend_a ? db : da) == 0) { term = 3; break; }
        // orient: reduce "u" (dividend) by "v" (divisor)
        uint32_t* wu = dividend_a ? wa : wb;
        const uint32_t* wv = dividend_a ? wb : wa;
        int& uu = dividend_a ? ua : ub;
        const int uv = dividend_a ? ub : ua;
        int& limu = dividend_a ? limA : limB;
        const int limv = dividend_a ? limB : limA;
        const int delta = uu - uv;
        const uint32_t x = wu[uu], y = wv[uv], negx = negmod(x, F);
        const int nlim = min(limu, limv + delta);
        for (int j = uu + lane; j < nlim; j += 32) wu[j] = ff_comb(y, wu[j], negx, wv[j - delta], F);
        // matrix rows: u-row (P11,P12 or P21,P22) -= shift(v-row, delta)
        const int ru = dividend_a ? 0 : 2, rv = dividend_a ? 2 : 0;
        __syncwarp();
        p_update(P + (ru + 0) * PL, lo[ru + 0], hi[ru + 0], P + (rv + 0) * PL, lo[rv + 0],
                 hi[rv + 0], delta, y, negx, W, F, err);
        p_update(P + (ru + 1) * PL, lo[ru + 1], hi[ru + 1], P + (rv + 1) * PL, lo[rv + 1],
                 hi[rv + 1], delta, y, negx, W, F, err);
        if (err) break;
        ++steps;
        limu = nlim;
        const int nu = first_nonzero(wu, uu + 1, nlim);
        int64_t& du = dividend_a ? da : db;
        const int64_t d0 = dividend_a ? da0 : db0;
        if (nu >= 0) {
            uu = nu;
            du = d0 - nu;
        } else if (d0 - (nlim - 1) <= 0) {
            uu = nlim;  // every word down to index 0 is zero: the operand vanished
            du = -1;
        } else {
            uu = nlim;  // the valid window ran out before a nonzero word
            du = d0 - nlim;
            unknown = true;
        }
    }
    if (lane == 0) {
        c.da0 = da0;
        c.db0 = db0;
        c.da1 = da;
        c.db1 = db;
        for (int i = 0; i < 4; ++i) {
            c.lo[i] = lo[i];
            c.hi[i] = hi[i];
        }
        c.steps = steps;
        c.term = term;
        c.dividend_a = dividend_a;
        c.err = err;
    }
}

// Z1[x] = sum_{d in [lo1,hi1]} P1[d] Z0[x+d] + sum_{d in [lo2,hi2]} P2[d] V0[x+sh+d]
// for x in [xs, xe): the matrix row applied by one CTA (all threads).
__device__ void apply_row(uint32_t* out, int64_t xs, int64_t xe, const uint32_t* P1, int lo1,
                          int hi1, const uint32_t* Z0, int64_t zb, const uint32_t* P2, int lo2,
                          int hi2, const uint32_t* V0, int64_t vb, int64_t sh, uint32_t* sw,
                          uint32_t* sv, int ORG, int W, const FieldParams& F) {
    constexpr int R = GCD_R;
    const int64_t n = xe - xs;
    if (n <= 0) return;
    for (int64_t c0 = 0; c0 < n; c0 += int64_t(GCD_T) * R) {
        const int64_t cn = i64min(n - c0, int64_t(GCD_T) * R);
        uint64_t acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0;
        uint32_t since = 0;
        for (int term = 0; term < 2; ++term) {
            const uint32_t* Pt = term ? P2 : P1;
            const int lo = term ? lo2 : lo1, hi = term ? hi2 : hi1;
            if (lo > hi) continue;
            const uint32_t* Zt = term ? V0 : Z0;
            const int64_t zbound = term ? vb : zb;
            const int64_t off = xs + c0 + (term ? sh : 0) + hi - ORG;  // sv[y] = Zt[y + off]
            const int width = hi - lo + 1, wpad = (width + R - 1) / R * R;
            __syncthreads();
            for (int u = threadIdx.x; u < wpad; u += GCD_T) sw[u] = u < width ? Pt[hi - u + W] : 0u;
            for (int64_t y = threadIdx.x; y < ORG + cn + R; y += GCD_T) {
                const int64_t x = y + off;
                sv[y] = (x >= 0 && x <= zbound) ? __ldcg(Zt + x) : 0u;
            }
            __syncthreads();
            const int64_t y0 = int64_t(threadIdx.x) * R;
            if (y0 < cn) conv_accumulate<R>(acc, sw, wpad / R, sv, int(ORG + y0), since, F);
        }
        const int64_t y0 = int64_t(threadIdx.x) * R;
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (y0 + r < cn) __stcg(out + xs + c0 + y0 + r, reduce(acc[r], F));
    }
}

}  // namespace

__global__ void __launch_bounds__(GCD_T) gcd_kernel(GcdArgs g) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ GcdCtl ctl;
    cg::grid_group grid = cg::this_grid();
    const int W = g.W, PL = 2 * W + 1;
    const FieldParams F = g.F;
    const int ORG = ((PL + 3) & ~3) + 3 + 4;
    const int64_t span = int64_t(GCD_T) * GCD_R;
    uint32_t* wa = smem;
    uint32_t* wb = wa + ((W + 3) & ~3);
    uint32_t* P = wb + ((W + 3) & ~3);
    uint32_t* sw = P + ((4 * PL + 3) & ~3);
    uint32_t* sv = sw + ((PL + 3 + 4) & ~3);

    const int64_t tid = int64_t(blockIdx.x) * GCD_T + threadIdx.x;
    const int64_t nthreads = int64_t(gridDim.x) * GCD_T;
    for (int64_t i = tid; i < g.na; i += nthreads) g.X[0][i] = g.a[i];
    for (int64_t i = tid; i < g.nb; i += nthreads) g.Y[0][i] = g.b[i];
    if (threadIdx.x == 0) {
        ctl.da1 = g.na - 1;
        ctl.db1 = g.nb - 1;
        ctl.dividend_a = 1;  // oracle_gcd: x = a is the first dividend (oracle.cpp:70)
        ctl.term = 0;
        ctl.err = 0;
    }
    grid.sync();

    int cur = 0;
    for (;;) {
        if (threadIdx.x < 32) run_chain(ctl, wa, wb, P, g, g.X[cur], g.Y[cur]);
        __syncthreads();
        if (ctl.err || (ctl.steps == 0 && ctl.term == 0)) {
            // internal invariant broken: report through the length word
            if (blockIdx.x == 0 && threadIdx.x == 0) *g.ng = ctl.err ? -1 : -2;
            return;  // grid-uniform decision: every CTA exits here
        }
        if (ctl.term == 3) break;
        if (ctl.steps > 0) {
            // apply the batch matrix: outputs A1[0..da1], B1[0..db1]
            const int64_t na1 = ctl.da1 + 1 > 0 ? ctl.da1 + 1 : 0;
            const int64_t nb1 = ctl.db1 + 1 > 0 ? ctl.db1 + 1 : 0;
            const int64_t per = (na1 + nb1 + gridDim.x - 1) / gridDim.x;
            const int64_t s0 = int64_t(blockIdx.x) * per, s1 = i64min(s0 + per, na1 + nb1);
            const int64_t da0 = ctl.da0, db0 = ctl.db0;
            // A part of this CTA's slice of [A1 | B1]
            apply_row(g.X[cur ^ 1], i64min(s0, na1), i64min(s1, na1), P + 0 * PL, ctl.lo[0],
                      ctl.hi[0], g.X[cur], da0, P + 1 * PL, ctl.lo[1], ctl.hi[1], g.Y[cur], db0,
                      db0 - da0, sw, sv, ORG, W, F);
            apply_row(g.Y[cur ^ 1], i64max(s0 - na1, 0), i64max(s1 - na1, 0), P + 3 * PL,
                      ctl.lo[3], ctl.hi[3], g.Y[cur], db0, P + 2 * PL, ctl.lo[2], ctl.hi[2],
                      g.X[cur], da0, da0 - db0, sw, sv, ORG, W, F);
            (void)span;
            grid.sync();
            cur ^= 1;
        }
        if (ctl.term) break;
    }
    // finalize: monic of the surviving operand, or 1
    __syncthreads();
    if (ctl.term == 3) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            g.g[0] = 1u;
            *g.ng = 1;
        }
        return;
    }
    const uint32_t* Z = ctl.term == 1 ? g.Y[cur] : g.X[cur];
    const int64_t dz = ctl.term == 1 ? ctl.db1 : ctl.da1;
    const uint32_t inv = invmod(__ldcg(Z + dz), F);
    for (int64_t i = tid; i <= dz; i += nthreads) g.g[i] = mulmod(__ldcg(Z + i), inv, F);
    if (blockIdx.x == 0 && threadIdx.x == 0) *g.ng = dz + 1;
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
    g.S = int(std::min<int64_t>(s, 1024));
    g.W = 2 * g.S + 32;
    g.cap = std::max<int64_t>(std::max(na, nb), 1);
    Scratch sc(st);
    for (int i = 0; i < 2; ++i) {
        g.X[i] = sc.get<uint32_t>(size_t(g.cap));
        g.Y[i] = sc.get<uint32_t>(size_t(g.cap));
    }
    const int W = g.W, PL = 2 * W + 1;
    const int ORG = ((PL + 3) & ~3) + 3 + 4;
    const size_t words = size_t(2 * ((W + 3) & ~3) + ((4 * PL + 3) & ~3) + ((PL + 3 + 4) & ~3) +
                                ORG + int64_t(GCD_T) * GCD_R + GCD_R + 8);
    const size_t bytes = words * 4;
    MMM_CUDA(cudaFuncSetAttribute(gcd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(bytes)));
    int per_sm = 0;
    MMM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gcd_kernel, GCD_T, bytes));
    if (per_sm < 1) throw Error(ST_INVALID, "gcd: s too large for shared memory");
    const int64_t want = std::max<int64_t>(1, ceil_div(na + nb, 512));
    const int blocks = int(std::min<int64_t>(want, int64_t(sm_count()) * per_sm));
    void* params[] = {&g};
    MMM_CUDA(cudaLaunchCooperativeKernel((void*)gcd_kernel, dim3(blocks), dim3(GCD_T), params, bytes,
                                         st));
    check_launch("gcd_kernel");
}

}  // namespace mmm_cu
