// divmod.cu -- long division over Z/pZ on sm_100a, s dividend heads per step.
//
// Replaces run_division (proj/src/division.cpp:81-176, Alg. 3-4)
// and computes exactly oracle_divmod (proj/src/oracle.cpp:51-67).
//
// The paper's optimized division retires s heads per launch; every block
// recomputes the s-head chain redundantly (division.cpp:127-138), one
// dependent modmul after another.  Here the chain is removed: with
//   h = rev(b)^-1 mod X^s            (power series, computed once),
// the s quotient words of one step are the truncated product
//   lambda_k = sum_{t<=k} h[k-t] * A[i-t],   k < s          (s^2/2 MACs)
// which is bit-identical to the sequential elimination, including the
// oracle's "skip a zero head" rule (a zero head yields lambda = 0).  The
// remainder update of the step,
//   A[x] -= sum_k lambda_k * b[x - i + k + db]   over the db words below,
// is the same register-tiled convolution as the product kernel (conv.cuh),
// and its b-window offset does not move between steps.
//
// Two schedules:
//   * div_cta_kernel  -- one CTA per instance, A and b resident in shared
//     memory, two CTA barriers per step (batched config, small instances);
//   * div_grid_kernel -- one persistent cooperative grid for a large single
//     instance: A stays in L2, each CTA owns a fixed slice of the db-long
//     active window relative to the heads and caches its b segment in shared
//     memory; one grid barrier per step of s heads (the paper's "launch").
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "conv.cuh"

namespace cg = cooperative_groups;

namespace mmm_cu {

// h[0..S) = rev(b)^-1 mod X^S, rev(b)_t = b[db - t].  One warp, S sequential
// coefficients, each a lane-parallel dot product.  bt(t) returns b[db - t].
template <class BT>
__device__ void inverse_series(uint32_t* h, int S, int64_t db, BT bt, const FieldParams& F) {
    const int lane = threadIdx.x & 31;
    const uint32_t h0 = invmod(bt(0), F);
    if (lane == 0) h[0] = h0;
    __syncwarp();
    const uint32_t nh0 = negmod(h0, F);
    for (int j = 1; j < S; ++j) {
        const int tmax = int(j < db ? j : db);
        uint64_t acc = 0;
        uint32_t since = 0;
        for (int t = 1 + lane; t <= tmax; t += 32) {
            if (++since > F.fold_terms) {
                acc = fold(acc, F);
                since = 1;
            }
            acc = mad_wide(bt(t), h[j - t], acc);
        }
        uint64_t v = reduce(acc, F);
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) h[j] = mulmod(reduce(v, F), nh0, F);
        __syncwarp();
    }
}

// lambda for one step: lam_rev[valid-1-k] = p - lambda_k  (negated, reversed,
// zero-padded to a multiple of R), write_q(k, lambda_k).  heads(t) = A[i-t].
template <class HD, class QW>
__device__ void step_lambdas(uint32_t* lam_rev, int valid, int padded, const uint32_t* h, HD heads,
                             QW write_q, const FieldParams& F) {
    for (int k = threadIdx.x; k < padded; k += blockDim.x) {
        uint32_t lam = 0;
        if (k < valid) {
            uint64_t acc = 0;
            uint32_t since = 0;
            for (int t = 0; t <= k; ++t) {
                if (++since > F.fold_terms) {
                    acc = fold(acc, F);
                    since = 1;
                }
                acc = mad_wide(h[k - t], heads(t), acc);
            }
            lam = reduce(acc, F);
            write_q(k, lam);
            lam_rev[valid - 1 - k] = negmod(lam, F);
        } else {
            lam_rev[k] = 0;
        }
    }
}

constexpr int DIV_T = 256;

struct DivArgs {
    const uint32_t* a;
    const uint32_t* b;
    uint32_t* q;
    uint32_t* r;
    int64_t na, nb, lda, ldb, ldq, ldr;
    int S;
    FieldParams F;
    Fan qf, rf;        // CTA kernel: q and r outputs (fan-out: every pointer gets the words)
    uint32_t* h_glob;  // grid kernel: inverse series
    uint32_t* a_work;  // grid kernel: working copy of A (L2 resident)
};

// ------------------------------------------------ one CTA per instance -----
// Shared layout (words): A[na] | bpad[BORG + nb + R] | h[S] | lam[Spad]
template <int R, bool FAN>
__global__ void __launch_bounds__(DIV_T) div_cta_kernel(DivArgs g, int borg) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int64_t inst = blockIdx.x;
    const int64_t na = g.na, nb = g.nb, db = nb - 1;
    const int S = g.S;
    const int Spad = (S + R - 1) / R * R;
    const FieldParams F = g.F;
    uint32_t* A = smem;
    uint32_t* bs = A + ((na + 3) & ~int64_t(3));  // bs[borg + j] = b[j], zero below
    uint32_t* h = bs + ((borg + nb + R + 3) & ~int64_t(3));
    uint32_t* lam = h + ((S + 3) & ~3);
    const uint32_t* a_g = g.a + inst * g.lda;
    const uint32_t* b_g = g.b + inst * g.ldb;
    const int64_t qbase = inst * g.ldq, rbase = inst * g.ldr;

    for (int64_t i = threadIdx.x; i < na; i += DIV_T) A[i] = a_g[i];
    for (int64_t j = threadIdx.x; j < borg + nb + R; j += DIV_T)
        bs[j] = (j >= borg && j < borg + nb) ? b_g[j - borg] : 0u;
    __syncthreads();
    if (threadIdx.x < 32)
        inverse_series(h, S, db, [&](int64_t t) { return t <= db ? bs[borg + db - t] : 0u; }, F);
    __syncthreads();

    for (int64_t i = na - 1; i >= db;) {
        const int valid = int(i - db + 1 < S ? i - db + 1 : S);
        const int padded = (valid + R - 1) / R * R;
        step_lambdas(lam, valid, padded, h, [&](int t) { return A[i - t]; },
                     [&](int k, uint32_t l) { fan_store<FAN>(g.qf, qbase + (i - db) - k, l); }, F);
        __syncthreads();
        const int64_t xlo = i - valid + 1 - db;  // update window [xlo, xlo + db)
        for (int64_t y0 = int64_t(threadIdx.x) * R; y0 < db; y0 += int64_t(DIV_T) * R) {
            uint64_t acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = (y0 + r < db) ? A[xlo + y0 + r] : 0u;
            uint32_t since = 0;
            conv_accumulate_auto<R>(acc, lam, padded / R, bs, int(borg + y0), since, F);
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (y0 + r < db) A[xlo + y0 + r] = reduce(acc[r], F);
        }
        __syncthreads();
        i -= valid;
    }
    for (int64_t x = threadIdx.x; x < db; x += DIV_T) fan_store<FAN>(g.rf, rbase + x, A[x]);
}

// ------------------------------------------- cooperative grid, 1 instance ---
// Per step of s heads: the heads are staged in shared memory with one
// coalesced load; the s quotient words are the truncated convolution
// lambda = h (*) heads computed by all threads with RL-word register tiles;
// the remainder update gives every thread RU outputs of this CTA's slice.
// Shared layout (words): bseg | hz (h, zero-padded below) | hd (heads) | lam
template <int RL, int RU>
__global__ void __launch_bounds__(DIV_T) div_grid_kernel(DivArgs g, int64_t seg) {
    extern __shared__ __align__(16) uint32_t smem[];
    cg::grid_group grid = cg::this_grid();
    const int64_t na = g.na, nb = g.nb, db = nb - 1;
    const int S = g.S;
    const int padL = (S + RL - 1) / RL * RL, padU = (S + RU - 1) / RU * RU;
    const FieldParams F = g.F;
    // this CTA's slice of the active window, relative to its bottom: [y_lo, y_hi)
    const int64_t y_lo = int64_t(blockIdx.x) * seg;
    const int64_t y_hi = y_lo + seg < db ? y_lo + seg : db;
    const int borg = ((padU + 3) & ~3) + 3;       // bseg[borg + (y - y_lo)] = b[y]
    const int horg = ((padL + 3) & ~3) + 3;       // hz[horg + j] = h[j], 0 for j < 0
    uint32_t* bseg = smem;
    const int64_t blen = borg + seg + RU + 1;
    uint32_t* hz = bseg + ((blen + 3) & ~int64_t(3));
    uint32_t* hd = hz + ((horg + padL + 8 + 3) & ~3);
    uint32_t* lam = hd + ((padL + 3) & ~3);
    uint32_t* A = g.a_work;

    for (int64_t j = threadIdx.x; j < blen; j += DIV_T) {
        const int64_t y = y_lo + j - borg;
        bseg[j] = (y >= 0 && y < nb) ? g.b[y] : 0u;
    }
    for (int64_t i = int64_t(blockIdx.x) * DIV_T + threadIdx.x; i < na;
         i += int64_t(gridDim.x) * DIV_T)
        A[i] = g.a[i];
    if (blockIdx.x == 0 && threadIdx.x < 32)
        inverse_series(g.h_glob, S, db,
                       [&](int64_t t) { return t <= db ? __ldcg(g.b + (db - t)) : 0u; }, F);
    grid.sync();
    for (int k = threadIdx.x; k < horg + padL + 8; k += DIV_T)
        hz[k] = (k >= horg && k - horg < S) ? __ldcg(g.h_glob + (k - horg)) : 0u;
    __syncthreads();

    for (int64_t i = na - 1; i >= db;) {
        const int valid = int(i - db + 1 < S ? i - db + 1 : S);
        const int nl = (valid + RL - 1) / RL * RL, nu = (valid + RU - 1) / RU * RU;
        for (int t = threadIdx.x; t < nl; t += DIV_T) hd[t] = t < valid ? __ldcg(A + (i - t)) : 0u;
        for (int t = valid + threadIdx.x; t < nu; t += DIV_T) lam[t] = 0u;
        __syncthreads();
        // lambda_k = sum_{t<=k} h[k-t] * A[i-t]   (k < valid)
        for (int k0 = int(threadIdx.x) * RL; k0 < valid; k0 += DIV_T * RL) {
            uint64_t acc[RL];
#pragma unroll
            for (int r = 0; r < RL; ++r) acc[r] = 0;
            uint32_t since = 0;
            conv_accumulate_auto<RL>(acc, hd, nl / RL, hz, horg + k0, since, F);
#pragma unroll
            for (int r = 0; r < RL; ++r) {
                const int k = k0 + r;
                if (k < valid) {
                    const uint32_t l = reduce(acc[r], F);
                    lam[valid - 1 - k] = negmod(l, F);
                    if (blockIdx.x == 0) g.q[i - db - k] = l;
                }
            }
        }
        __syncthreads();
        const int64_t xlo = i - valid + 1 - db;
        for (int64_t y0 = y_lo + int64_t(threadIdx.x) * RU; y0 < y_hi;
             y0 += int64_t(DIV_T) * RU) {
            uint64_t acc[RU];
#pragma unroll
            for (int r = 0; r < RU; ++r) acc[r] = (y0 + r < y_hi) ? __ldcg(A + xlo + y0 + r) : 0u;
            uint32_t since = 0;
            conv_accumulate_auto<RU>(acc, lam, nu / RU, bseg, int(borg + (y0 - y_lo)), since, F);
#pragma unroll
            for (int r = 0; r < RU; ++r)
                if (y0 + r < y_hi) __stcg(A + xlo + y0 + r, reduce(acc[r], F));
        }
        grid.sync();
        i -= valid;
    }
    for (int64_t x = int64_t(blockIdx.x) * DIV_T + threadIdx.x; x < db;
         x += int64_t(gridDim.x) * DIV_T)
        g.r[x] = __ldcg(A + x);
}

// ------------------------------------------- pipelined single instance --
// div_pipe_kernel: the large single division without a grid barrier per step.
// Steps j = 0..J-1 retire the heads [i_j - v_j + 1, i_j] (v_j = S but the
// last), i_j = max(na - 1 - j*S, db - 1).  The step's update
//   A[x] += sum_{k<v} nl_k * b[x - i_j + db + k],   nl_k = -lambda_k,
// depends only on the step's lambdas, so updates commute and may be applied
// to different positions at different times.  CTA 0 (head) keeps the top
// WH = 2S positions of A in shared memory, computes each step's lambdas from
// its window (split-K tiled convolution with h = rev(b)^-1), publishes them
// as tagged words (lam_t: no flag, no fence), updates its window and the
// S positions entering it, then slides.  Entering positions come from global
// A, where the bulk CTAs have applied every step up to j - L; the head adds
// the last L steps from its lambda history.  Bulk CTAs own fixed blocks of
// PIPE_B positions (round robin) and apply published steps k to positions
// x <= i_{k+L} - WH, several steps per pass; each publishes its progress.
// The head waits only for the owners of its entering positions, L steps
// behind.  Result: identical to the grid kernel (and the oracle).
#ifdef PIPE_DBG_NOCONV  // timing experiments only (tools/head_bench.cu)
#define PIPE_CONV(x) (void)0
#else
#define PIPE_CONV(x) x
#endif
// Bulk lag (steps the head absorbs): the kernel is instantiated for the split
// head's lag (DIV_PIPE_L, 2: best measured for it) and the M-form head's
// (DIV_PIPE_LM, 4: its cheaper steps leave room for a longer hand-off).
#ifndef DIV_PIPE_L
#define DIV_PIPE_L 2
#endif
#ifndef DIV_PIPE_LM
#define DIV_PIPE_LM 4
#endif
#ifndef DIV_PIPE_CT
#define DIV_PIPE_CT 256
#endif
constexpr int PIPE_CT = DIV_PIPE_CT;  // compute threads of the head (8 warps: A 4, B 4)
constexpr int PIPE_T = PIPE_CT + 32;  // + the head's control warp
constexpr int PIPE_B = PIPE_CT;       // positions per bulk block
constexpr int PIPE_MAXB = 4;    // steps per bulk pass

struct PipeArgs {
    const uint32_t* a;
    const uint32_t* b;
    uint32_t* q;
    uint32_t* r;
    int64_t na, nb;
    int S;
    FieldParams F;
    uint32_t* A;            // working copy of the dividend (L2 resident)
    uint32_t* h_glob;       // inverse series (S words)
    uint64_t* lam_t;        // step k's negated lambdas, tagged (k + 1) << 32 | value: J * S words
    unsigned* progress;     // per bulk CTA: steps applied to all of its blocks
    long long* stats;       // optional (MMM_DIV_STATS): cycle counters
    bool b_smem;            // bulk CTAs hold all of b in shared memory
    bool mform;             // head: pipe_head_m (S = 128, odd p, fold_terms >= 16)
};

namespace {

__device__ __forceinline__ void bar_sync_n(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// Tagged words (tag << 32 | value), single-copy-atomic 64-bit relaxed accesses:
// a reader polls the word it needs until it carries the expected tag, so the
// lambdas reach the bulk CTAs with no flag and no fence (a release store on the
// head's SM measured ~8k cycles).
__device__ __forceinline__ void pipe_st_tag(uint64_t* p, uint32_t v, unsigned tag) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"((uint64_t(tag) << 32) | v)
                 : "memory");
}
__device__ __forceinline__ uint64_t pipe_ld_rlx64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t pipe_ld_tag(const uint64_t* p, unsigned tag) {
    uint64_t w;
    while (unsigned((w = pipe_ld_rlx64(p)) >> 32) != tag) {
    }
    return uint32_t(w);
}
// Publishing after a CTA barrier: the barrier orders the CTA's writes before
// the publishing thread's release store, which is cumulative at gpu scope
// (the pattern of CUTLASS's semaphore release).  A __threadfence() before it
// compiles to MEMBAR.SC.GPU (~1 us measured); DIV_PIPE_SCFENCE=1 restores it.
#ifndef DIV_PIPE_SCFENCE
#define DIV_PIPE_SCFENCE 0
#endif
__device__ __forceinline__ void pipe_sc_fence() {
#if DIV_PIPE_SCFENCE
    __threadfence();
#endif
}
__device__ __forceinline__ void pipe_st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Origin of h in the head's zero-padded copy: a lambda part reads up to
// SPANL - 1 + 3 words below it (SPANL <= max(64, S / 2)).
__host__ __device__ constexpr int pipe_horg(int S) {
    return ((S / 2 + 3) & ~3) + 3 > 67 ? ((S / 2 + 3) & ~3) + 3 : 67;
}

// i(k): the top of step k's heads (db - 1 once all steps are done)
__device__ __forceinline__ int64_t pipe_i(int64_t na, int64_t db, int S, int64_t k) {
    const int64_t v = na - 1 - k * S;
    return v > db - 1 ? v : db - 1;
}

// v[k] = the reduced sum over the quad's P parts (adjacent lanes, P a power
// of two <= 32) of accumulator k, on every part's lane.  Lane `part` then
// stores the words r = part, part + P, ... < 4 of the quad.
__device__ __forceinline__ void quad_reduce(uint64_t (&acc)[4], int P, uint32_t (&v)[4],
                                            const FieldParams& F) {
#ifdef PIPE_DBG_NOREDUCE  // timing experiments only (tools/head_bench.cu)
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = uint32_t(acc[k]);
    return;
#endif
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = reduce(acc[k], F);
    for (int d = 1; d < P; d <<= 1)
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = addmod(v[k], __shfl_xor_sync(0xffffffffu, v[k], d), F);
}

// Split-K tiled sum with the parts across warps and the quads across lanes:
// item it -> (quad it % NQ, part it / NQ), so a warp's lanes hold consecutive
// quads of one part (shared-memory reads broadcast or consecutive: no bank
// conflicts) and the parts meet in a shared-memory reduction (red: P x 4*NQ
// words) instead of a lane butterfly.  item(qd, part, acc) adds the part's
// terms for the quad's 4 outputs; store(t, v) receives output t < 4*NQ.
template <class Item, class Store>
__device__ __forceinline__ void tiled_sum(int NQ, int P, uint32_t* red, Item item, Store store,
                                          const FieldParams& F, int nthreads, int barid,
                                          int tid) {
    const int NO = 4 * NQ;
    for (int it = tid; it < NQ * P; it += nthreads) {
        const int part = it / NQ, qd = it - part * NQ;
        uint64_t acc[4] = {0, 0, 0, 0};
        item(qd, part, acc);
#pragma unroll
        for (int r = 0; r < 4; ++r) red[part * NO + 4 * qd + r] = reduce(acc[r], F);
    }
    bar_sync_n(barid, nthreads);
    for (int t = tid; t < NO; t += nthreads) {
        uint64_t sum = 0;
        for (int p = 0; p < P; ++p) sum += red[p * NO + t];
        store(t, reduce(sum, F));
    }
}

}  // namespace

// pipe_head_split: the same head with its compute warps in two groups, so the
// entering update leaves the per-step critical path.  Step j's lambdas need
// the heads (window [0, S) after step j-1); the window update of step j
// (positions [v, 2S)) feeds step j+1's heads; the entering words of step j
// (positions [2S, 2S + v), steps j-1 and j on top of the bulk's) are needed
// only by step j+1's window update.  Group A (DIV_PIPE_AW warps) runs
// lambda -> window; group B (the other compute warps) runs entering_j
// concurrently with A's window_j and lambda_{j+1}.  Hand-offs are named
// barriers with arrive (producer) / sync (consumer), by step parity:
//   LAM(j): A's lambda_j written        -> B and the control warp
//   ENT(j): B's entering_j in the window -> A, before window_{j+1}
//   STG(j): control staged E_j          -> B
// The lambda history is a ring of L + 1 steps (B reads j-1 and j while A
// writes j+1).  Same arithmetic, same result as pipe_head.
#ifndef DIV_PIPE_AW
#define DIV_PIPE_AW 4
#endif
template <int L>
__device__ void pipe_head_split(const PipeArgs& g, uint32_t* sm, int nbulk) {
    constexpr int LR = L + 1, CT = PIPE_CT;
    constexpr int AT = 32 * DIV_PIPE_AW, BT = CT - AT;
    static_assert(L >= 1 && AT > 0 && BT > 0, "pipe_head_split: both groups non-empty");
    constexpr int BAR_A = 1, BAR_B = 2, BAR_LAM = 3, BAR_ENT = 5, BAR_STG = 7;
    const FieldParams F = g.F;
    const int S = g.S, tid = threadIdx.x, WH = 2 * S, WR = 4 * S;
    const int logS = 31 - __clz(S);
    const int64_t na = g.na, db = g.nb - 1;
    const int64_t J = (na - db + S - 1) / S;
    const bool control = tid >= CT, groupA = tid < AT;
    const int horg = pipe_horg(S);
    uint32_t* hz = sm;                                   // h at hz[horg + m]
    uint32_t* hd = hz + ((horg + S + 8 + 3) & ~3);      // heads, S words
    uint32_t* lamh = hd + S;                             // LR x S negated lambdas
    uint32_t* win = lamh + LR * S;                       // ring by absolute position
    uint32_t* stage = win + WR;                          // 2 x S entering words
    uint32_t* bt3 = stage + 2 * S;                       // bt3[3 + m] = b[db - m]
    const int MB = (L + 2) * S + 16;
    uint32_t* redA = bt3 + ((MB + 3) & ~3);              // tiled_sum partials, 4 * AT words
    uint32_t* redB = redA + 4 * AT;                      // 4 * BT words
    for (int m = tid; m < horg + S + 8; m += PIPE_T) {
        const int j = m - horg;
        hz[m] = (j >= 0 && j < S) ? __ldcg(g.h_glob + j) : 0u;
    }
    for (int m = tid; m < MB; m += PIPE_T) {
        const int64_t x = db - (m - 3);
        bt3[m] = (m >= 3 && x >= 0) ? g.b[x] : 0u;
    }
    for (int m = tid; m < LR * S; m += PIPE_T) lamh[m] = 0u;
    const int64_t i0 = na - 1;
    for (int t = tid; t < WH; t += PIPE_T) {
        const int64_t x = i0 - t;
        win[x & (WR - 1)] = x >= 0 ? __ldcg(g.A + x) : 0u;
    }
    long long c_poll = 0;
    auto stage_entering = [&](int64_t jj) {
        const int64_t hi = pipe_i(na, db, S, jj) - WH, lo = pipe_i(na, db, S, jj + 1) - WH + 1;
        if (hi < 0 || hi < lo) return;
        const int lane = tid & 31;
        const int64_t need = jj - L + 1;
        if (lane < 2 && need > 0) {
            const int64_t x = lane == 0 ? (lo > 0 ? lo : 0) : hi;
            const int owner = int((x / PIPE_B) % nbulk);
            const long long cp = clock64();
            spin_until_geq(g.progress + owner, unsigned(need));  // acquire load, no MEMBAR
#ifdef PIPE_DBG_FAKE_POLL  // timing experiments only (tools/head_bench.cu): a bulk round trip
            while (clock64() - cp < PIPE_DBG_FAKE_POLL) {
            }
#endif
            c_poll += clock64() - cp;
        }
        __syncwarp();
        uint32_t* st = stage + (jj & 1) * S;
        for (int64_t x = lo + lane; x <= hi; x += 32) st[x - lo] = x >= 0 ? __ldcg(g.A + x) : 0u;
    };
    if (control) stage_entering(0);
    __syncthreads();
    long long c_loop = clock64(), c_pub = 0, c_stage = 0, c_lam = 0, c_win = 0, c_ent = 0,
              c_wait = 0;
    if (control) {
        for (int64_t j = 0; j < J; ++j) {
            bar_sync_n(BAR_LAM + int(j & 1), PIPE_T);
            const long long c1 = clock64();
            if (j + 1 < J) {
                stage_entering(j + 1);
                bar_arrive_n(BAR_STG + int((j + 1) & 1), BT + 32);
            }
            c_stage += clock64() - c1;
        }
    } else if (groupA) {
        int PL = 1;  // lambda tiling: S/4 quads x PL parts over the S head terms
        while ((S / 4) * PL * 2 <= AT && PL * 2 <= S / 4) PL *= 2;
        const int SPANL = S / PL;
        for (int64_t j = 0; j < J; ++j) {
            const int64_t i = pipe_i(na, db, S, j), inext = pipe_i(na, db, S, j + 1);
            const int v = int(i - inext);
            const long long p0 = clock64();
            for (int t = tid; t < S; t += AT) hd[t] = t < v ? win[(i - t) & (WR - 1)] : 0u;
            bar_sync_n(BAR_A, AT);
            uint32_t* lj = lamh + int(j % LR) * S;
            tiled_sum(
                S / 4, PL, redA,
                [&](int qd, int part, uint64_t (&acc)[4]) {
                    const int k0 = 4 * qd, t0 = part * SPANL;
                    uint32_t since = 0;
                    if (t0 <= k0 + 3)
                        PIPE_CONV(conv_accumulate4_fast(acc, hd + t0, SPANL / 4, hz, horg + k0 - t0,
                                                        since, F));
                },
                [&](int k, uint32_t lam) {
                    const uint32_t nl = k < v ? negmod(lam, F) : 0u;
                    if (k < v) {
                        g.q[i - db - k] = lam;
                        pipe_st_tag(g.lam_t + j * S + k, nl, unsigned(j + 1));
                    }
                    lj[k] = nl;
                },
                F, AT, BAR_A, tid);
            bar_arrive_n(BAR_LAM + int(j & 1), PIPE_T);
            const long long p1 = clock64();
            c_lam += p1 - p0;
            // E_{j-1} complete; either barrier also orders group A's lambda stores (lj)
            // before the window pass reads them -- at j = 0 nothing else did, and a
            // delayed warp (another kernel sharing the SM) then updated the window with
            // stale zeros: step 0's quotient right, every later word wrong
            if (j >= 1)
                bar_sync_n(BAR_ENT + int((j - 1) & 1), CT);
            else
                bar_sync_n(BAR_A, AT);
            const long long p2 = clock64();
            c_wait += p2 - p1;
            // window (t in [v, WH)): step j
            const int tq = v & ~3, NQ = (WH - tq) >> 2, vp = (v + 3) & ~3;
            int P = 1;
            while (NQ * P * 2 <= AT && (S / (P * 2)) >= 4 && ((S / (P * 2)) & 3) == 0) P *= 2;
            const int SPAN = S / P;
            tiled_sum(
                NQ, P, redA,
                [&](int qd, int part, uint64_t (&acc)[4]) {
                    const int t0 = tq + 4 * qd, k0 = part * SPAN;
                    uint32_t since = 0;
                    if (k0 < vp)
                        PIPE_CONV(conv_accumulate4_fast(acc, lj + k0, min(SPAN, vp - k0) / 4, bt3,
                                                        t0 - k0 + 3, since, F));
                },
                [&](int tt, uint32_t add) {
                    const int t = tq + tt;
                    const int64_t x = i - t;
                    if (t >= v && t < WH && x >= 0) {
                        uint32_t* w = win + (x & (WR - 1));
                        *w = addmod(*w, add, F);
                    }
                },
                F, AT, BAR_A, tid);
            bar_sync_n(BAR_A, AT);
            c_win += clock64() - p2;
        }
        if (J >= 1) bar_sync_n(BAR_ENT + int((J - 1) & 1), CT);  // the last entering words
    } else {
        const int tb = tid - AT;
        for (int64_t j = 0; j < J; ++j) {
            const int64_t i = pipe_i(na, db, S, j), inext = pipe_i(na, db, S, j + 1);
            const int v = int(i - inext);
            const long long p0 = clock64();
            bar_sync_n(BAR_LAM + int(j & 1), PIPE_T);                // lambda_j
            if (j >= 1) bar_sync_n(BAR_STG + int(j & 1), BT + 32);  // E_j staged
            const long long p1 = clock64();
            c_wait += p1 - p0;
            // entering (t in [WH, WH + v)): stage + steps j - 1 .. j
            const uint32_t* st = stage + (j & 1) * S;
            const int NQ = (v + 3) >> 2, TT = L * S;
            int P = 1;
            while (NQ * P * 2 <= BT && (TT / (P * 2)) >= 4 && ((TT / (P * 2)) & 3) == 0) P *= 2;
            const int SPAN = TT / P;
            tiled_sum(
                NQ, P, redB,
                [&](int qd, int part, uint64_t (&acc)[4]) {
                    const int t0 = WH + 4 * qd;
                    uint32_t since = 0;
                    for (int c0 = part * SPAN; c0 < (part + 1) * SPAN;) {
                        const int d = c0 >> logS, k0 = c0 & (S - 1);
                        const int n = min(S - k0, (part + 1) * SPAN - c0);
                        const int lim = d == 0 ? ((v + 3) & ~3) : S;
                        if (j - d >= 0 && k0 < lim)
                            PIPE_CONV(conv_accumulate4_fast(acc, lamh + int((j - d) % LR) * S + k0,
                                                            min(n, lim - k0) / 4, bt3,
                                                            t0 + d * S - k0 + 3, since, F));
                        c0 += n;
                    }
                },
                [&](int tt, uint32_t add) {
                    const int t = WH + tt;
                    const int64_t x = i - t;
                    if (tt < v && x >= 0) win[x & (WR - 1)] = addmod(st[v - 1 - tt], add, F);
                },
                F, BT, BAR_B, tb);
            bar_arrive_n(BAR_ENT + int(j & 1), CT);
            c_ent += clock64() - p1;
        }
    }
    if (g.stats && tid == 0) {
        g.stats[0] = J;
        g.stats[1] = clock64() - c_loop;
        g.stats[8] = c_lam;
        g.stats[9] = c_win;
        g.stats[11] = c_wait;
    }
    if (g.stats && tid == AT) {
        g.stats[10] = c_ent;
        g.stats[3] = c_wait;
    }
    if (g.stats && tid == CT) {
        g.stats[2] = c_stage;
        g.stats[4] = c_poll;
    }
    (void)c_pub;
    __syncthreads();
    for (int t = tid; t < WH; t += PIPE_T) {
        const int64_t x = (db - 1) - t;
        if (x >= 0) __stcg(g.A + x, win[x & (WR - 1)]);
    }
}

// pipe_head_m: the head with one product per step on its chain (S = 128).
// With Z_j = step j's heads before step j-1's update (steps <= j-2 applied)
// and the step's negated lambdas nl_j = -lambda_j,
//   lambda_j = T_h Z_j + Mb nl_{j-1},
//   Mb[r][k] = sum_{t <= r} h[r - t] b[db - S - t + k]   (T_h: lower-triangular
//   Toeplitz of h; Mb: step j-1's update of step j's heads, solved by T_h),
// and Z_{j+2} is exactly step j's entering words (positions [2S, 3S) below
// step j's top, steps <= j applied).  So the old chain -- lambda_j, then the
// window update that forms step j+1's heads -- becomes one pass: Mb sits in
// the compute threads' registers (a 4 x 16 block each, Montgomery form, built
// once by a diagonal walk Mb[r][k] = Mb[r-1][k-1] + h[r] b[db - S + k]), the
// window is never materialised, and after the last step the top 2S remainder
// words are formed from the last Z's and lambdas.  All eight compute warps run
// the chain and then the entering words; the control warp stages as before.
constexpr int PIPE_HS_OFF = 16384;  // head: h computed here (words; the head layout ends below)
constexpr int MF_S = 128;
constexpr int MST_OFF = PIPE_HS_OFF + 512;  // the walk's staging of Mb (S x S words)
template <int L>
__device__ void pipe_head_m(const PipeArgs& g, uint32_t* sm, int nbulk) {
    constexpr int S = MF_S, LR = L + 1, CT = PIPE_CT, WH = 2 * S;
    constexpr int logS = 7;
    static_assert(CT == 256 && L >= 2 && L <= 4, "pipe_head_m: eight compute warps, lag 2..4");
    constexpr int BAR_C = 1, BAR_LAM = 3, BAR_STG = 7;  // LAM / STG by step parity
    constexpr int MB = (L + 2) * S + 16;
    const FieldParams F = g.F;
    const int tid = threadIdx.x;
    const int64_t na = g.na, db = g.nb - 1;
    const int64_t J = (na - db + S - 1) / S;
    const bool control = tid >= CT;
    uint32_t* hz = sm;                // hz[S + m] = h[m], zeros around
    uint32_t* lamh = hz + 2 * S + 8;  // LR x S negated lambdas, ring by step
    uint32_t* stage = lamh + LR * S;  // 2 x S entering words (control warp)
    uint32_t* bt3 = stage + 2 * S;    // bt3[3 + m] = b[db - m]
    uint32_t* Zr = bt3 + MB;          // 3 x S: Z_j in slot j % 3
    uint32_t* part = Zr + 3 * S;      // 8 x S chain partials
    uint32_t* red = part + 8 * S;     // tiled_sum partials (8 x 4 x 32)
    uint32_t* tmpu = red + 1024;      // S
    uint32_t* bw = tmpu + S;          // S: b[db - S + k] 2^64 mod p
    uint32_t* bx = bw + S;            // bx[m] = b[db - m], m < (L+2) S (16-byte aligned windows)
    uint32_t* Mst = sm + MST_OFF;
    for (int m = tid; m < 2 * S + 8; m += PIPE_T) {
        const int j = m - S;
        hz[m] = (j >= 0 && j < S) ? __ldcg(g.h_glob + j) : 0u;
    }
    for (int m = tid; m < MB; m += PIPE_T) {
        const int64_t x = db - (m - 3);
        bt3[m] = (m >= 3 && x >= 0) ? g.b[x] : 0u;
        if (m >= 3 && m < (L + 2) * S + 3) bx[m - 3] = (x >= 0) ? g.b[x] : 0u;
    }
    for (int m = tid; m < LR * S; m += PIPE_T) lamh[m] = 0u;
    {  // Z_0 and Z_1: the top 2S words, no step applied
        const int64_t i0 = na - 1;
        for (int t = tid; t < WH; t += PIPE_T) {
            const int64_t x = i0 - t;
            Zr[t] = x >= 0 ? __ldcg(g.A + x) : 0u;  // slot 0 = Z_0, slot 1 = Z_1
        }
    }
    long long c_poll = 0;
    auto stage_entering = [&](int64_t jj) {  // as in pipe_head_split
        const int64_t hi = pipe_i(na, db, S, jj) - WH, lo = pipe_i(na, db, S, jj + 1) - WH + 1;
        if (hi < 0 || hi < lo) return;
        const int lane = tid & 31;
        const int64_t need = jj - L + 1;
        if (need > 0) {  // the whole warp polls the owners of both ends
            const int64_t x = (lane & 1) == 0 ? (lo > 0 ? lo : 0) : hi;
            const unsigned* pw = g.progress + int((x / PIPE_B) % nbulk);
            const long long cp = clock64();
#ifndef PIPE_DBG_NOSPIN  // timing experiments: no wait for the bulk (wrong results)
            while (__any_sync(0xffffffffu, ld_relaxed_gpu(pw) < unsigned(need))) {
            }
            (void)spin_until_geq(pw, unsigned(need));  // the acquiring load
#endif
            c_poll += clock64() - cp;
        }
        __syncwarp();
        uint32_t* st = stage + (jj & 1) * S;
        for (int64_t x = lo + lane; x <= hi; x += 32) st[x - lo] = x >= 0 ? __ldcg(g.A + x) : 0u;
    };
    if (control) stage_entering(0);
    __syncthreads();
    long long c_loop = clock64(), c_mv = 0, c_ent = 0, c_wait = 0, c_build = 0, c_ts = 0;
    if (control) {
        for (int64_t j = 0; j < J; ++j) {
            bar_sync_n(BAR_LAM + int(j & 1), PIPE_T);
            if (j + 1 < J) {
                stage_entering(j + 1);
                bar_arrive_n(BAR_STG + int((j + 1) & 1), PIPE_T);
            }
        }
    } else {
        const long long cb = clock64();
        // ---- Mb in Montgomery form (x 2^32), by a diagonal walk through Mst ----
        if (tid < S) {
            bw[tid] = reduce_odd(uint64_t(bt3[3 + S - tid]) * F.r2, F);  // b[db - S + k] R^2
            uint64_t u = 0;  // Mb[r][0] = sum_{t <= r} h[r - t] b[db - S - t]
            uint32_t since = 0;
            for (int t = 0; t <= tid; ++t) {
                if (++since > F.fold_terms) {
                    u = fold(u, F);
                    since = 1;
                }
                u = mad_wide(hz[S + tid - t], bt3[3 + S + t], u);
            }
            tmpu[tid] = reduce_odd(uint64_t(reduce_odd(u, F)) * F.r2, F);
        }
        bar_sync_n(BAR_C, CT);
        auto at = [](int r, int k) { return r * S + (k ^ (((r >> 2) & 7) << 2)); };
        {
            const int dl = tid - 127;
            if (dl < 128) {
                const int r = dl >= 0 ? dl : 0, k = dl >= 0 ? 0 : -dl;
                uint64_t acc = dl >= 0 ? uint64_t(tmpu[dl]) : uint64_t(hz[S]) * bw[k];
                Mst[at(r, k)] = redc(fold(acc, F), F);
                const int len = 128 - (dl >= 0 ? dl : -dl);
                acc = fold(acc, F);
                int i = 1;
                for (; i + 16 <= len; i += 16) {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        acc = mad_wide(hz[S + r + i + q], bw[k + i + q], acc);
                        Mst[at(r + i + q, k + i + q)] = redc(fold(acc, F), F);
                    }
                    acc = fold(acc, F);
                }
                for (; i < len; ++i) {
                    acc = mad_wide(hz[S + r + i], bw[k + i], acc);
                    Mst[at(r + i, k + i)] = redc(fold(acc, F), F);
                }
            }
        }
        bar_sync_n(BAR_C, CT);
        const int gq = tid & 31, pq = tid >> 5;
        uint32_t mm[4][16], hw[19];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const uint4 w4 = *reinterpret_cast<const uint4*>(
                    Mst + (4 * gq + k) * S + ((16 * pq + 4 * jj) ^ ((gq & 7) << 2)));
                mm[k][4 * jj] = w4.x;
                mm[k][4 * jj + 1] = w4.y;
                mm[k][4 * jj + 2] = w4.z;
                mm[k][4 * jj + 3] = w4.w;
            }
#pragma unroll
        for (int i = 0; i < 19; ++i) hw[i] = hz[S + 4 * gq - 16 * pq - 15 + i];
        bar_sync_n(BAR_C, CT);
        c_build = clock64() - cb;
        // ring slots kept incrementally (no 64-bit modulo per step): Z by j % 3, the
        // lambda history by j % LR
        int r0 = 0, l0 = 0;
        for (int64_t j = 0; j < J; ++j, r0 = r0 == 2 ? 0 : r0 + 1, l0 = l0 == LR - 1 ? 0 : l0 + 1) {
            const int rp2 = r0 == 0 ? 2 : r0 - 1;                   // (j + 2) % 3
            const int lm1 = l0 == 0 ? LR - 1 : l0 - 1;              // (j - 1) % LR
            const int64_t i = pipe_i(na, db, S, j), inext = pipe_i(na, db, S, j + 1);
            const int v = int(i - inext);
            const long long p0 = clock64();
            // ---- the chain: lambda_j = T_h Z_j + Mb nl_{j-1} ----
            {
                const uint32_t* zj = Zr + r0 * S + 16 * pq;
                const uint32_t* np = lamh + lm1 * S + 16 * pq;  // zeros at j = 0
                uint32_t z[16], q[16];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const uint4 zv = *reinterpret_cast<const uint4*>(zj + 4 * c);
                    const uint4 qv = *reinterpret_cast<const uint4*>(np + 4 * c);
                    z[4 * c] = zv.x; z[4 * c + 1] = zv.y; z[4 * c + 2] = zv.z; z[4 * c + 3] = zv.w;
                    q[4 * c] = qv.x; q[4 * c + 1] = qv.y; q[4 * c + 2] = qv.z; q[4 * c + 3] = qv.w;
                }
                uint64_t a1[4] = {0, 0, 0, 0}, a2[4] = {0, 0, 0, 0};
#pragma unroll
                for (int jj = 0; jj < 16; ++jj)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        a1[k] = mad_wide(hw[k - jj + 15], z[jj], a1[k]);
                        a2[k] = mad_wide(mm[k][jj], q[jj], a2[k]);
                    }
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    part[pq * S + 4 * gq + k] = reduce_odd(a1[k], F) + redc(fold(a2[k], F), F);
            }
            bar_sync_n(BAR_C, CT);
            if (tid < S) {
                uint64_t sum = 0;
#pragma unroll
                for (int pp = 0; pp < 8; ++pp) sum += part[pp * S + tid];
                const uint32_t lam = reduce_odd(sum, F);
                const int k = tid;
                const uint32_t nl = k < v ? negmod(lam, F) : 0u;
                if (k < v) {
                    g.q[i - db - k] = lam;
                    pipe_st_tag(g.lam_t + j * S + k, nl, unsigned(j + 1));
                }
                lamh[l0 * S + k] = nl;
            }
            bar_sync_n(BAR_C, CT);
            bar_arrive_n(BAR_LAM + int(j & 1), PIPE_T);
            const long long p1 = clock64();
            c_mv += p1 - p0;
            if (j >= 1) bar_sync_n(BAR_STG + int(j & 1), PIPE_T);  // E_j staged
            const long long p2 = clock64();
            c_wait += p2 - p1;
            // ---- entering_j -> Z_{j+2}: stage + steps j - 1 .. j ----
            // value[tt] = st + sum_{d<L} sum_k nl_{j-d}[k] b[db - (2S + tt + dS - k)]: thread
            // (gq, pq) takes rows 4gq..4gq+3 and the 16 L combined terms c in
            // [16 L pq, +16 L) (c = dS + k), b in a sliding register window (16-byte loads
            // from bx), 16 terms per chunk
            {
                uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
                for (int hh = 0; hh < L; ++hh) {
                    const int c = 16 * L * pq + 16 * hh, d = c >> logS, k0 = c & (S - 1);
                    const int ld = l0 - d < 0 ? l0 - d + LR : l0 - d;  // (j - d) % LR
                    const uint32_t* X = bx + 2 * S + d * S;           // X[i] = b[db - 2S - dS - i]
                    const uint32_t* W = lamh + ld * S + k0;           // nl_{j-d}[k0 ..]
                    uint32_t xw[20], wv[16];  // xw[i] = X[4gq - k0 - 16 + i]
#pragma unroll
                    for (int q4 = 0; q4 < 5; ++q4) {
                        const uint4 t4 = *reinterpret_cast<const uint4*>(X + 4 * gq - k0 - 16 + 4 * q4);
                        xw[4 * q4] = t4.x; xw[4 * q4 + 1] = t4.y; xw[4 * q4 + 2] = t4.z; xw[4 * q4 + 3] = t4.w;
                    }
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const uint4 t4 = *reinterpret_cast<const uint4*>(W + 4 * q4);
                        wv[4 * q4] = t4.x; wv[4 * q4 + 1] = t4.y; wv[4 * q4 + 2] = t4.z; wv[4 * q4 + 3] = t4.w;
                    }
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj)
#pragma unroll
                        for (int k = 0; k < 4; ++k)  // X[4gq + k - (k0 + jj)]
                            acc[k] = mad_wide(xw[k - jj + 16], wv[jj], acc[k]);
#pragma unroll
                    for (int k = 0; k < 4; ++k) acc[k] = fold(acc[k], F);  // 16 terms per chunk
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) part[pq * S + 4 * gq + k] = reduce_odd(acc[k], F);
                bar_sync_n(BAR_C, CT);
                if (tid < S) {
                    const int tt = tid;
                    uint64_t sum = 0;
#pragma unroll
                    for (int pp = 0; pp < 8; ++pp) sum += part[pp * S + tt];
                    const uint32_t add = reduce_odd(sum, F);
                    const uint32_t* st = stage + (j & 1) * S;
                    const int64_t x = i - WH - tt;
                    if (tt < v) Zr[rp2 * S + tt] = x >= 0 ? addmod(st[v - 1 - tt], add, F) : 0u;
                }
            }
            c_ts += clock64() - p2;
            bar_sync_n(BAR_C, CT);
            c_ent += clock64() - p2;
        }
        // ---- the top 2S remainder words below the last heads (x = db - 1 - t) ----
        // t < S - v: Z_{J-1}[t + v] + steps J-2, J-1;  t < 2S - v: Z_J[t - S + v] + step
        // J-1;  else Z_{J+1}[t - 2S + v] (every step applied)
        {
            const int64_t iJ1 = pipe_i(na, db, S, J - 1);
            const int v = int(iJ1 - (db - 1));
            const int t = tid;  // 2S outputs, one per compute thread
            const int64_t x = db - 1 - t;
            const uint32_t* n1 = lamh + int((J - 1) % LR) * S;  // (zero-initialised slots:
            const uint32_t* n2 = lamh + int((J - 2) % LR) * S;  //  J >= 3 here)
            auto bb = [&](int m) { return m < 0 ? 0u : bt3[3 + m]; };  // b[db - m]
            uint32_t base;
            int steps;
            if (t < S - v) {
                base = Zr[int((J - 1) % 3) * S + t + v];
                steps = 2;
            } else if (t < 2 * S - v) {
                base = Zr[int(J % 3) * S + t - S + v];
                steps = 1;
            } else {
                base = Zr[int((J + 1) % 3) * S + t - 2 * S + v];
                steps = 0;
            }
            uint64_t acc = 0;
            uint32_t since = 0;
            if (steps >= 1)
                for (int kk = 0; kk < S; ++kk) {  // step J-1: b[db - (t + v) + kk]
                    if (++since > F.fold_terms) {
                        acc = fold(acc, F);
                        since = 1;
                    }
                    acc = mad_wide(n1[kk], bb(t + v - kk), acc);
                }
            if (steps >= 2)
                for (int kk = 0; kk < S; ++kk) {  // step J-2: b[db - (t + v + S) + kk]
                    if (++since > F.fold_terms) {
                        acc = fold(acc, F);
                        since = 1;
                    }
                    acc = mad_wide(n2[kk], bb(t + v + S - kk), acc);
                }
            if (x >= 0) __stcg(g.A + x, addmod(base, reduce_odd(acc, F), F));
        }
    }
    if (g.stats && tid == 0) {
        g.stats[0] = J;
        g.stats[1] = clock64() - c_loop;
        g.stats[8] = c_mv;
        g.stats[9] = c_build;
        g.stats[10] = c_ent;
        g.stats[11] = c_wait;
        g.stats[3] = c_ts;
    }
    if (g.stats && tid == CT) g.stats[4] = c_poll;
    if (g.stats && tid == 33) g.stats[2] = c_ts;
    __syncthreads();
}

// Bulk shared layout (words): lam [PIPE_MAXB * S + 4] | bw [PIPE_B + S + 8,
// padded] | bz [nb + 2 * PIPE_PADB] when the whole divisor fits (g.b_smem):
// bz[PIPE_PADB + x] = b[x], zero outside [0, db], loaded once per launch, so
// a step's b window is a shared-memory copy instead of an L2 round trip.
constexpr int PIPE_PADB = PIPE_B + 264;
__host__ __device__ constexpr int64_t pipe_bulk_words(int S, int64_t nb, bool b_smem) {
    return int64_t(PIPE_MAXB) * S + 4 + ((PIPE_B + S + 8 + 3) & ~3) + 4 * PIPE_B +
           (b_smem ? nb + 2 * PIPE_PADB : 0);
}


__device__ void pipe_bulk_load_b(const PipeArgs& g, uint32_t* sm) {
    if (!g.b_smem) return;
    uint32_t* bz = sm + PIPE_MAXB * g.S + 4 + ((PIPE_B + g.S + 8 + 3) & ~3) + 4 * PIPE_B;
    const int64_t n = g.nb + 2 * PIPE_PADB, db = g.nb - 1;
#pragma unroll 8
    for (int64_t y = threadIdx.x; y < n; y += PIPE_T) {
        const int64_t x = y - PIPE_PADB;
        bz[y] = (x >= 0 && x <= db) ? __ldcg(g.b + x) : 0u;
    }
}

template <int L>
__device__ void pipe_bulk(const PipeArgs& g, uint32_t* sm, int nbulk, int me) {
    const FieldParams F = g.F;
    const int S = g.S, tid = threadIdx.x, WH = 2 * S;
    const int64_t na = g.na, db = g.nb - 1;
    const int64_t J = (na - db + S - 1) / S;
    const int64_t nblocks = (na + PIPE_B - 1) / PIPE_B;  // every position below the heads
    uint32_t* lam = sm;                          // per step of the pass: S reversed negated lambdas
    uint32_t* bw = lam + PIPE_MAXB * S + 4;      // b window: PIPE_B + S + 8 words
    uint32_t* red = bw + ((PIPE_B + S + 8 + 3) & ~3);  // 4 parts x PIPE_B partial sums
    uint32_t* bz = red + 4 * PIPE_B;
    const bool b_smem = g.b_smem;  // bz loaded by pipe_bulk_load_b before the grid barrier
    __shared__ unsigned pub_s;
    // 4 positions per thread, 4 parts over the step's terms: PIPE_B/4 x 4 = the
    // first PIPE_B threads (whole warps; the ninth warp only stages and syncs).
    // A warp's lanes hold consecutive quads of one part (16-byte window reads of
    // consecutive words: no bank conflicts); the parts meet in shared memory.
    static_assert(PIPE_B == PIPE_CT, "pipe_bulk: one quad x part per compute thread");
    const bool worker = tid < PIPE_B;
    const int part = tid / (PIPE_B / 4), qd = tid % (PIPE_B / 4);
    long long c_wait = 0, c_work = 0, passes = 0, c_rel = 0, c_lam = 0;
    int64_t k = 0;
    while (k < J) {
        const long long tw = clock64();
        if (tid == 0) {  // step k's first lambda carries its tag; later steps: no wait
            pipe_ld_tag(g.lam_t + k * S, unsigned(k + 1));
            int64_t e = k + 1;
            while (e < J && e < k + PIPE_MAXB &&
                   unsigned(pipe_ld_rlx64(g.lam_t + e * S) >> 32) == unsigned(e + 1))
                ++e;
            pub_s = unsigned(e);
        }
        __syncthreads();
        const long long tb = clock64();
        c_wait += tb - tw;
        ++passes;
        const int64_t kend = min(int64_t(pub_s), k + int64_t(PIPE_MAXB));
        const long long tl = clock64();
        // the pass's lambdas, once for all blocks: lam[(kk - k) * S + u] = nl_{v-1-u}
        for (int64_t kk = k; kk < kend; ++kk) {
            const int64_t ik = pipe_i(na, db, S, kk);
            const int v = int(ik - pipe_i(na, db, S, kk + 1)), vp = (v + 3) & ~3;
            uint32_t* lk = lam + (kk - k) * S;
            for (int u = tid; u < vp; u += PIPE_T) {
                const int kp = v - 1 - u;
                lk[u] = kp >= 0 ? pipe_ld_tag(g.lam_t + kk * S + kp, unsigned(kk + 1)) : 0u;
            }
        }
        if (tid == 0) c_lam += clock64() - tl;
        __syncthreads();  // the pass's lambdas in
        for (int64_t beta = me; beta < nblocks; beta += nbulk) {
            const int64_t blo = beta * PIPE_B, bhi = min(blo + int64_t(PIPE_B), na);
            const int64_t x0 = blo + 4 * qd;
            // this thread's stored position (blo + tid), loaded ahead: only this CTA writes it
            const uint32_t a_old = (worker && blo + tid < bhi) ? __ldcg(g.A + blo + tid) : 0u;
            uint64_t acc[4] = {0, 0, 0, 0};  // sum of per-step canonical partials
            bool touched = false;
            for (int64_t kk = k; kk < kend; ++kk) {
                const int64_t ik = pipe_i(na, db, S, kk);
                const int64_t v = ik - pipe_i(na, db, S, kk + 1);
                const int64_t xlo = ik - v + 1 - db;
                const int64_t top = min(pipe_i(na, db, S, kk + L) - int64_t(WH), ik - v);
                if (bhi - 1 < xlo || blo > top) continue;  // uniform over the CTA
                touched = true;
                const int vp = int((v + 3) & ~3);
                const int64_t bwlo = blo - ik + db + v - vp;  // window[y] = b[bwlo + y]
                // b in shared memory at the window's alignment: read it in place (no copy,
                // no barrier); otherwise stage the window
                const bool direct = b_smem && ((PIPE_PADB + bwlo) & 3) == 0;
                const uint32_t* win = direct ? bz + PIPE_PADB + bwlo : bw;
                if (!direct) {
                    __syncthreads();  // previous step's window consumed
                    if (b_smem) {
                        for (int y = tid; y < PIPE_B + vp + 8; y += PIPE_T) bw[y] = bz[PIPE_PADB + bwlo + y];
                    } else {
                        for (int y = tid; y < PIPE_B + vp + 8; y += PIPE_T) {
                            const int64_t bx = bwlo + y;
                            bw[y] = (bx >= 0 && bx <= db) ? __ldcg(g.b + bx) : 0u;
                        }
                    }
                    __syncthreads();
                }
                // part's terms: [u0, u0 + n), multiples of 4
                const int span = ((vp / 4 + 3) & ~3) > 4 ? ((vp / 4 + 3) & ~3) : 4;
                const int u0 = part * span;
                if (worker && u0 < vp) {
                    uint64_t pa[4] = {0, 0, 0, 0};
                    uint32_t since = 0;
                    conv_accumulate4_fast(pa, lam + (kk - k) * S + u0, min(span, vp - u0) / 4, win,
                                          4 * qd + vp - 1 - u0, since, F);
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int64_t xr = x0 + r;
                        if (xr >= xlo && xr <= top && xr < bhi) acc[r] += reduce(pa[r], F);
                    }
                }
            }
            if (!touched) continue;  // (uniform over the CTA)
            if (worker)
#pragma unroll
                for (int r = 0; r < 4; ++r) red[part * PIPE_B + 4 * qd + r] = reduce(acc[r], F);
            __syncthreads();
            if (worker) {
                // position blo + tid: the four parts' sums; store only positions a step
                // updated (the rest may belong to the head, whose final words must not
                // be overwritten by a late pass)
                const int64_t xp = blo + tid;
                bool upd = false;
                for (int64_t kk = k; kk < kend; ++kk) {
                    const int64_t ik = pipe_i(na, db, S, kk);
                    const int64_t v = ik - pipe_i(na, db, S, kk + 1);
                    const int64_t top = min(pipe_i(na, db, S, kk + L) - int64_t(WH), ik - v);
                    if (xp >= ik - v + 1 - db && xp <= top) upd = true;
                }
                if (upd && xp < bhi) {
                    const uint64_t sum = uint64_t(red[tid]) + red[PIPE_B + tid] +
                                         red[2 * PIPE_B + tid] + red[3 * PIPE_B + tid];
                    __stcg(g.A + xp, addmod(a_old, reduce(sum, F), F));
                }
            }
            // the partial sums are read: the next block's may be written (with b read
            // in place nothing else separates the two; uniform over the CTA)
            if (beta + nbulk < nblocks) __syncthreads();
        }
        __syncthreads();
        const long long tr = clock64();
        if (tid == 0) {
            pipe_sc_fence();
            pipe_st_release(g.progress + me, unsigned(kend));
        }
        c_rel += clock64() - tr;
        c_work += clock64() - tb;
        k = kend;
    }
    if (g.stats && me == 0 && tid == 0) {
        g.stats[5] = c_wait;
        g.stats[6] = c_work;
        g.stats[7] = passes;
        g.stats[12] = c_rel;
        g.stats[13] = c_lam;
    }
}

template <int L>
__global__ void __launch_bounds__(PIPE_T, 1) div_pipe_kernel(PipeArgs g) {
    extern __shared__ __align__(16) uint32_t smem[];
    cg::grid_group grid = cg::this_grid();
    const int64_t na = g.na, db = g.nb - 1;
    for (int64_t i = int64_t(blockIdx.x) * PIPE_T + threadIdx.x; i < na;
         i += int64_t(gridDim.x) * PIPE_T)
        g.A[i] = g.a[i];
    // Before the grid barrier: the head's warp 0 computes h in shared memory
    // (each coefficient reads the earlier ones: an L2 round trip apiece if h
    // lived in global memory) and publishes it; the bulk CTAs load b.
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        uint32_t* hs = smem + PIPE_HS_OFF;
        inverse_series(hs, g.S, db,
                       [&](int64_t t) { return t <= db ? __ldcg(g.b + (db - t)) : 0u; }, g.F);
        for (int t = threadIdx.x; t < g.S; t += 32) g.h_glob[t] = hs[t];
    } else if (blockIdx.x > 0) {
        pipe_bulk_load_b(g, smem);
    }
    grid.sync();
    const int nbulk = gridDim.x - 1;
    if (blockIdx.x == 0 && g.mform)
        pipe_head_m<L>(g, smem, nbulk);
    else if (blockIdx.x == 0)
        pipe_head_split<L>(g, smem, nbulk);
    else
        pipe_bulk<L>(g, smem, nbulk, blockIdx.x - 1);
    grid.sync();
    for (int64_t x = int64_t(blockIdx.x) * PIPE_T + threadIdx.x; x < db;
         x += int64_t(gridDim.x) * PIPE_T)
        g.r[x] = __ldcg(g.A + x);
}

// ------------------------------------------ division by a constant (nb = 1) --
// oracle_divmod with deg b = 0 (oracle.cpp:51-67): every head i yields
// lambda = r[i] * lc(b)^-1, q[i] = lambda, and r[i] -= lambda * b[0] leaves 0,
// so q = a * b[0]^-1 and r = 0 (the zero-head skip gives the same q[i] = 0).
// Grid (chunks, instances); one inverse per CTA.
template <bool FAN>
__global__ void __launch_bounds__(256) div_const_kernel(const uint32_t* __restrict__ A, int64_t lda,
                                                        int64_t na, const uint32_t* __restrict__ B,
                                                        int64_t ldb, Fan Q, int64_t ldq,
                                                        FieldParams F) {
    __shared__ uint32_t cinv;
    const int64_t inst = blockIdx.y;
    if (threadIdx.x == 0) cinv = invmod(B[inst * ldb], F);
    __syncthreads();
    const uint32_t c = cinv;
    const uint32_t* a = A + inst * lda;
    const int64_t qb = inst * ldq;
    for (int64_t j = int64_t(blockIdx.x) * 256 + threadIdx.x; j < na; j += int64_t(gridDim.x) * 256)
        fan_store<FAN>(Q, qb + j, mulmod(__ldg(a + j), c, F));
}

namespace {

void run_const(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
               const uint32_t* B, int64_t ldb, int64_t count, Fan Q, int64_t ldq,
               cudaStream_t st) {
    const int64_t per = std::max<int64_t>(1, std::min<int64_t>(ceil_div(na, 256),
                                                               ceil_div(8LL * sm_count(), count)));
    for (int64_t c0 = 0; c0 < count; c0 += 65535) {
        const unsigned n = unsigned(std::min<int64_t>(65535, count - c0));
        const dim3 grid(unsigned(std::min<int64_t>(per, 65535)), n);
        const Fan q = fan_offset(Q, c0 * ldq);
        if (Q.n > 1)
            div_const_kernel<true><<<grid, 256, 0, st>>>(A + c0 * lda, lda, na, B + c0 * ldb, ldb,
                                                         q, ldq, F);
        else
            div_const_kernel<false><<<grid, 256, 0, st>>>(A + c0 * lda, lda, na, B + c0 * ldb, ldb,
                                                          q, ldq, F);
        check_launch("div_const_kernel", grid, dim3(256));
    }
}

int pick_R(const FieldParams& F) { return F.fold_terms >= 8 ? 8 : (F.fold_terms >= 2 ? 2 : 1); }

size_t cta_smem_words(int64_t na, int64_t nb, int S, int R, int borg) {
    const int Spad = (S + R - 1) / R * R;
    return size_t(((na + 3) & ~3) + ((borg + nb + R + 3) & ~3) + ((S + 3) & ~3) + Spad + 4);
}

template <int R>
void run_cta(const DivArgs& g, int64_t count, cudaStream_t st) {
    const int Spad = (g.S + R - 1) / R * R;
    const int borg = ((Spad + 3) & ~3) + 3;
    const size_t bytes = cta_smem_words(g.na, g.nb, g.S, R, borg) * 4;
    const bool fan = g.qf.n > 1 || g.rf.n > 1;
    auto kern = fan ? div_cta_kernel<R, true> : div_cta_kernel<R, false>;
    MMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(bytes)));
    for (int64_t c0 = 0; c0 < count; c0 += 65535) {
        DivArgs gg = g;
        gg.a += c0 * g.lda;
        gg.b += c0 * g.ldb;
        gg.qf = fan_offset(g.qf, c0 * g.ldq);
        gg.rf = fan_offset(g.rf, c0 * g.ldr);
        const unsigned n = unsigned(std::min<int64_t>(65535, count - c0));
        kern<<<n, DIV_T, bytes, st>>>(gg, borg);
        check_launch("div_cta_kernel", dim3(n), dim3(DIV_T));
    }
}

template <int RL, int RU>
void run_grid(DivArgs g, cudaStream_t st) {
    const int S = g.S;
    const int padL = (S + RL - 1) / RL * RL, padU = (S + RU - 1) / RU * RU;
    const int64_t db = g.nb - 1;
    int per_sm = 0;
    // slice per CTA: a full pass of the CTA's threads, at most one CTA per SM
    const int ctas_max = sm_count();
    int64_t seg = std::max<int64_t>(ceil_div(db, ctas_max), int64_t(DIV_T) * RU);
    seg = ceil_div(seg, RU) * RU;
    const int borg = ((padU + 3) & ~3) + 3, horg = ((padL + 3) & ~3) + 3;
    const int64_t blen = borg + seg + RU + 1;
    const size_t words = size_t(((blen + 3) & ~int64_t(3)) + ((horg + padL + 8 + 3) & ~3) +
                                ((padL + 3) & ~3) + padU + 8);
    const size_t bytes = words * 4;
    MMM_CUDA(cudaFuncSetAttribute(div_grid_kernel<RL, RU>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    MMM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, div_grid_kernel<RL, RU>,
                                                           DIV_T, bytes));
    const int64_t blocks = ceil_div(db, seg);
    if (per_sm < 1 || blocks > int64_t(per_sm) * ctas_max)
        throw Error(ST_SIM, "division: grid does not fit co-resident");
    Scratch sc(st);
    g.h_glob = sc.get<uint32_t>(size_t(S));
    g.a_work = sc.get<uint32_t>(size_t(g.na));
    void* params[] = {&g, &seg};
    MMM_CUDA(cudaLaunchCooperativeKernel((void*)div_grid_kernel<RL, RU>, dim3(unsigned(blocks)),
                                         dim3(DIV_T), params, bytes, st));
    check_launch("div_grid_kernel", dim3(unsigned(blocks)), dim3(DIV_T));
}

// Pipelined schedule (div_pipe_kernel): S = s rounded down to a power of two
// in [32, 256] (the result does not depend on S); needs 4 products per fold.
bool pipe_eligible(const FieldParams& F, int64_t s) { return s >= 32 && F.fold_terms >= 8; }

void run_pipe(const DivArgs& d, int64_t s, cudaStream_t st) {
    int S = 32;
    while (S * 2 <= s && S < 256) S *= 2;
    PipeArgs g{};
    g.a = d.a;
    g.b = d.b;
    g.q = d.q;
    g.r = d.r;
    g.na = d.na;
    g.nb = d.nb;
    g.S = S;
    g.F = d.F;
    const int64_t Jm = (d.na - (d.nb - 1) + S - 1) / S;
    g.mform = S == MF_S && d.F.odd && d.F.fold_terms >= 16 && Jm >= 3 && !getenv("MMM_DIV_PIPE_OLD");
    const int L = g.mform ? DIV_PIPE_LM : DIV_PIPE_L;
    auto kern = g.mform ? div_pipe_kernel<DIV_PIPE_LM> : div_pipe_kernel<DIV_PIPE_L>;
    const int horg = pipe_horg(S);
    const size_t head =
        size_t(((horg + S + 8 + 3) & ~3) + S + (L + 1) * S + 4 * S + 2 * S + (L + 2) * S + 16 + 4 * PIPE_CT);
    g.b_smem = pipe_bulk_words(S, d.nb, true) * 4 <= 220 * 1024 && !getenv("MMM_DIV_BULK_GLOBAL_B");
    const size_t bulk = size_t(pipe_bulk_words(S, d.nb, g.b_smem));
    // more than half an SM's shared memory: one CTA per SM, so no bulk CTA
    // shares (and takes issue slots from) the head's SM
    const size_t head_m = g.mform ? size_t(MST_OFF + MF_S * MF_S) : 0;
    const size_t bytes = std::max<size_t>(
        std::max(std::max(std::max(head, bulk), head_m), size_t(PIPE_HS_OFF + S)) * 4, 120 * 1024);
    MMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    int per_sm = 0;
    MMM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PIPE_T, bytes));
    if (per_sm < 1) throw Error(ST_SIM, "division: pipelined grid does not fit");
    // one CTA per SM (the head's SM to itself), no more bulk CTAs than blocks
    const int blocks = int(std::min<int64_t>(sm_count(), 1 + ceil_div(d.na, PIPE_B)));
    Scratch sc(st);
    g.A = sc.get<uint32_t>(size_t(d.na));
    g.h_glob = sc.get<uint32_t>(size_t(S));
    g.progress = sc.get<unsigned>(size_t(blocks));
    MMM_CUDA(cudaMemsetAsync(g.progress, 0, size_t(blocks) * sizeof(unsigned), st));
    const int64_t J = (d.na - (d.nb - 1) + S - 1) / S;
    g.lam_t = sc.get<uint64_t>(size_t(J) * S);  // tags start at 1: zeroed words never match
    MMM_CUDA(cudaMemsetAsync(g.lam_t, 0, size_t(J) * S * sizeof(uint64_t), st));
    const bool want_stats = getenv("MMM_DIV_STATS") != nullptr;
    if (want_stats) {
        g.stats = sc.get<long long>(16);
        MMM_CUDA(cudaMemsetAsync(g.stats, 0, 16 * sizeof(long long), st));
    }
    void* params[] = {&g};
    MMM_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(unsigned(blocks)), dim3(PIPE_T), params,
                                         bytes, st));
    check_launch("div_pipe_kernel", dim3(unsigned(blocks)), dim3(PIPE_T));
    if (want_stats) {
        long long h[16];
        MMM_CUDA(cudaMemcpyAsync(h, g.stats, sizeof(h), cudaMemcpyDeviceToHost, st));
        MMM_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr,
                "div pipe stats: S=%d blocks=%d steps=%lld head_loop=%lld ctl_stage=%lld "
                "B_wait=%lld (ctl poll=%lld) | hd+lambda=%lld (waitA=%lld) window=%lld "
                "entering=%lld | bulk0 wait=%lld work=%lld passes=%lld release=%lld lambdas=%lld\n",
                S, blocks, h[0], h[1], h[2], h[3], h[4], h[8], h[11], h[9], h[10], h[5], h[6],
                h[7], h[12], h[13]);
    }
}

}  // namespace

void launch_divmod(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b,
                   int64_t nb, uint32_t* q, uint32_t* r, int64_t s, cudaStream_t st) {
    if (s < 1) throw Error(ST_INVALID, "division: block parameter must be >= 1");
    const int64_t mu = na - nb + 1;
    const int S = int(std::min<int64_t>(std::min<int64_t>(s, mu), 4096));
    DivArgs g{};
    g.a = a;
    g.b = b;
    g.q = q;
    g.r = r;
    g.qf = fan_of(q);
    g.rf = fan_of(r);
    g.na = na;
    g.nb = nb;
    g.S = S;
    g.F = F;
    const int R = pick_R(F);
    const int Spad = (S + R - 1) / R * R;
    const int borg = ((Spad + 3) & ~3) + 3;
    const size_t cta_bytes = cta_smem_words(na, nb, S, R, borg) * 4;
    if (nb == 1) {  // division by a constant: q = a * b[0]^-1, no remainder words
        run_const(F, a, na, na, b, 1, 1, g.qf, 0, st);
        return;
    }
    const bool small = double(mu) * double(nb) < 4.0e6 && cta_bytes <= 200 * 1024;
    if (small) {
        switch (R) {
            case 8: run_cta<8>(g, 1, st); break;
            case 2: run_cta<2>(g, 1, st); break;
            default: run_cta<1>(g, 1, st); break;
        }
        return;
    }
    // the pipeline keeps 2S remainder words and S entering words per step in
    // its head: divisors shorter than that take the grid schedule
    const char* force = getenv("MMM_DIV_SCHED");  // tests/tools: "grid" or "pipe"
    const bool want_pipe = force ? std::string(force) == "pipe"
                                 : (nb > 4 * 256 && !getenv("MMM_DIV_GRID"));
    if (pipe_eligible(F, s) && want_pipe) {
        run_pipe(g, s, st);
        return;
    }
    switch (R) {
        case 8: run_grid<4, 2>(g, st); break;
        case 2: run_grid<2, 2>(g, st); break;
        default: run_grid<1, 1>(g, st); break;
    }
}

void launch_divmod_batched(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                           const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, uint32_t* Q,
                           int64_t ldq, uint32_t* Rr, int64_t ldr, int64_t s, cudaStream_t st) {
    launch_divmod_batched_fan(F, A, lda, na, B, ldb, nb, count, fan_of(Q), ldq, fan_of(Rr), ldr, s,
                              st);
}

void launch_divmod_batched_fan(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                               const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, Fan Q,
                               int64_t ldq, Fan Rr, int64_t ldr, int64_t s, cudaStream_t st) {
    if (nb >= 2 && tcdiv_supported(na, nb, count, s)) {  // 128 heads per step on the tensor core
        launch_tcdiv_batched(F, A, lda, na, B, ldb, nb, count, Q, ldq, Rr, ldr, st);
        return;
    }
    if (s <= 0) s = 64;  // auto on the CUDA cores
    if (s < 1) throw Error(ST_INVALID, "division: block parameter must be >= 1");
    const int64_t mu = na - nb + 1;
    DivArgs g{};
    g.a = A;
    g.b = B;
    g.qf = Q;
    g.rf = Rr;
    g.na = na;
    g.nb = nb;
    g.lda = lda;
    g.ldb = ldb;
    g.ldq = ldq;
    g.ldr = ldr;
    g.S = int(std::min<int64_t>(std::min<int64_t>(s, mu), 4096));
    g.F = F;
    const int R = pick_R(F);
    const int Spad = (g.S + R - 1) / R * R;
    const int borg = ((Spad + 3) & ~3) + 3;
    if (nb == 1) {
        run_const(F, A, lda, na, B, ldb, count, Q, ldq, st);
        return;
    }
    if (cta_smem_words(na, nb, g.S, R, borg) * 4 > 200 * 1024) {
        // instances too large for one CTA: one single-instance division each
        // (grid or pipelined schedule), results fanned out by a copy kernel
        const int64_t lq = na - nb + 1, lr = nb - 1;
        for (int64_t i = 0; i < count; ++i) {
            Scratch sc(st);
            uint32_t* q = sc.get<uint32_t>(size_t(lq));
            uint32_t* r = sc.get<uint32_t>(size_t(lr));
            launch_divmod(F, A + i * lda, na, B + i * ldb, nb, q, r, s, st);
            launch_fanout_copy(q, lq, fan_offset(Q, i * ldq), st);
            launch_fanout_copy(r, lr, fan_offset(Rr, i * ldr), st);
        }
        return;
    }
    switch (R) {
        case 8: run_cta<8>(g, count, st); break;
        case 2: run_cta<2>(g, count, st); break;
        default: run_cta<1>(g, count, st); break;
    }
}

}  // namespace mmm_cu
