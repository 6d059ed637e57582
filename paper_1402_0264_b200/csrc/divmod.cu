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
// zero-padded to a multiple of R), q[i-db-k] = lambda_k.  heads(t) = A[i-t].
template <class HD>
__device__ void step_lambdas(uint32_t* lam_rev, int valid, int padded, const uint32_t* h, HD heads,
                             uint32_t* q_top, bool write_q, const FieldParams& F) {
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
            if (write_q) q_top[-k] = lam;
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
    uint32_t* h_glob;  // grid kernel: inverse series
    uint32_t* a_work;  // grid kernel: working copy of A (L2 resident)
};

// ------------------------------------------------ one CTA per instance -----
// Shared layout (words): A[na] | bpad[BORG + nb + R] | h[S] | lam[Spad]
template <int R>
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
    uint32_t* q_g = g.q + inst * g.ldq;
    uint32_t* r_g = g.r + inst * g.ldr;

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
        step_lambdas(lam, valid, padded, h, [&](int t) { return A[i - t]; }, q_g + (i - db), true,
                     F);
        __syncthreads();
        const int64_t xlo = i - valid + 1 - db;  // update window [xlo, xlo + db)
        for (int64_t y0 = int64_t(threadIdx.x) * R; y0 < db; y0 += int64_t(DIV_T) * R) {
            uint64_t acc[R];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = (y0 + r < db) ? A[xlo + y0 + r] : 0u;
            uint32_t since = 0;
            conv_accumulate<R>(acc, lam, padded / R, bs, int(borg + y0), since, F);
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (y0 + r < db) A[xlo + y0 + r] = reduce(acc[r], F);
        }
        __syncthreads();
        i -= valid;
    }
    for (int64_t x = threadIdx.x; x < db; x += DIV_T) r_g[x] = A[x];
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
            conv_accumulate<RL>(acc, hd, nl / RL, hz, horg + k0, since, F);
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
            conv_accumulate<RU>(acc, lam, nu / RU, bseg, int(borg + (y0 - y_lo)), since, F);
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

namespace {

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
    MMM_CUDA(cudaFuncSetAttribute(div_cta_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(bytes)));
    for (int64_t c0 = 0; c0 < count; c0 += 65535) {
        DivArgs gg = g;
        gg.a += c0 * g.lda;
        gg.b += c0 * g.ldb;
        gg.q += c0 * g.ldq;
        gg.r += c0 * g.ldr;
        const unsigned n = unsigned(std::min<int64_t>(65535, count - c0));
        div_cta_kernel<R><<<n, DIV_T, bytes, st>>>(gg, borg);
        check_launch("div_cta_kernel");
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
    check_launch("div_grid_kernel");
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
    g.na = na;
    g.nb = nb;
    g.S = S;
    g.F = F;
    const int R = pick_R(F);
    const int Spad = (S + R - 1) / R * R;
    const int borg = ((Spad + 3) & ~3) + 3;
    const size_t cta_bytes = cta_smem_words(na, nb, S, R, borg) * 4;
    const bool small = double(mu) * double(nb) < 4.0e6 && cta_bytes <= 200 * 1024;
    if (small || nb == 1) {
        if (cta_bytes > 200 * 1024) throw Error(ST_INVALID, "division: instance too large");
        switch (R) {
            case 8: run_cta<8>(g, 1, st); break;
            case 2: run_cta<2>(g, 1, st); break;
            default: run_cta<1>(g, 1, st); break;
        }
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
    if (s < 1) throw Error(ST_INVALID, "division: block parameter must be >= 1");
    const int64_t mu = na - nb + 1;
    DivArgs g{};
    g.a = A;
    g.b = B;
    g.q = Q;
    g.r = Rr;
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
    if (cta_smem_words(na, nb, g.S, R, borg) * 4 > 200 * 1024)
        throw Error(ST_INVALID, "division batch: instance too large for one CTA");
    switch (R) {
        case 8: run_cta<8>(g, count, st); break;
        case 2: run_cta<2>(g, count, st); break;
        default: run_cta<1>(g, count, st); break;
    }
}

}  // namespace mmm_cu
