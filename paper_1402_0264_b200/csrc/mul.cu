// mul.cu -- plain (schoolbook) multiplication over Z/pZ on sm_100a.
//
// Replaces the MUL + ADD kernel program of run_multiplication
// (proj/src/multiplication.cpp:23-164; Alg. 5-7) and computes the
// same product as oracle_mul (proj/src/oracle.cpp:8-15).
//
// Output-stationary 2-D tiling of the (k, i) parallelogram {0 <= i < na,
// 0 <= k - i < nb}: a CTA of MUL_T threads owns TK = MUL_T*R consecutive
// outputs ("k-tile") and one contiguous range of input indices i ("item"),
// staged through shared memory MUL_TI terms at a time; each thread keeps R
// outputs in 64-bit registers (conv.cuh).  The reference's M array of
// (x-1)*y partial rows and its log2 ADD rounds disappear: when a k-tile's
// i-range is split over several items, the items' reduced partial sums
// (< p each) meet in a 64-bit global accumulator through RED.ADD.64, and the
// last item to arrive on a k-tile reduces it (no second launch) -- the ADD
// rounds of the paper, done in L2 instead of log-round launches.  Batched
// products give each instance whole k-tiles (no split).  Chunks are double
// buffered through registers (cp.async at 4-byte granularity measured slower).
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "conv.cuh"

namespace mmm_cu {

constexpr int MUL_T = 128;   // threads per CTA
#ifndef MUL_GROUPED
#define MUL_GROUPED 1  // straight-line 32-term groups in the inner loop
#endif
#ifndef MUL_ARRIVE
#define MUL_ARRIVE 2  // split k-tile arrival: 1 = __threadfence + atomicAdd, 2 = one acq_rel atomic
#endif
#ifndef MUL_TI_WORDS
#define MUL_TI_WORDS 256
#endif
constexpr int MUL_TI = MUL_TI_WORDS;  // terms per shared-memory chunk

struct MulArgs {
    const uint32_t* a;
    const uint32_t* b;
    uint32_t* f;              // output word k - klo of instance inst at f[inst * ldf + k - klo]
    unsigned long long* acc;  // split k-tiles accumulate here (single instance)
    unsigned* arrived;        // per k-tile count of finished items
    // acc and arrived are the thread's ZeroBuf, all-zero between calls:
    // the last item of a k-tile reads its words and zeroes them (and resets
    // its counter), so no zeroing pass runs before the kernel
    int64_t na, nb, lda, ldb, ldf;
    int64_t chunk;  // i-range per item
    int64_t klo, khi;  // output range [klo, khi): f[k - klo] (whole product: 0, na + nb - 1)
    FieldParams F;
    Fan fan;  // fan-out instantiation: the same words into every fan.p[q] (fan.p[0] == f)
};

template <int R, bool FAN>
__global__ void __launch_bounds__(MUL_T) mul_kernel(MulArgs g) {
    constexpr int TK = MUL_T * R;
    constexpr int ORIGIN = MUL_TI + 3;  // == 3 (mod 4): aligned window reloads
    constexpr int SV = MUL_TI + TK + 4;
    constexpr int NW = (MUL_TI + MUL_T - 1) / MUL_T, NV = (SV + MUL_T - 1) / MUL_T;
    // two buffers: the next chunk is loaded into registers while this one is
    // multiplied, then written to the other buffer (one barrier per chunk)
    __shared__ __align__(16) uint32_t sw[2][MUL_TI];
    __shared__ __align__(16) uint32_t sv[2][SV];

    const int64_t inst = blockIdx.z;
    const uint32_t* __restrict__ a = g.a + inst * g.lda;
    const uint32_t* __restrict__ b = g.b + inst * g.ldb;
    const int64_t na = g.na, nb = g.nb, nf = g.khi;
    const int64_t k0 = g.klo + int64_t(blockIdx.y) * TK;
    if (k0 >= nf) return;
    const int64_t ilo = k0 - (nb - 1) > 0 ? k0 - (nb - 1) : 0;
    const int64_t ihi = k0 + TK < na ? k0 + TK : na;
    const int64_t i_begin = ilo + int64_t(blockIdx.x) * g.chunk;
    if (i_begin >= ihi) return;
    const int64_t i_end = i_begin + g.chunk < ihi ? i_begin + g.chunk : ihi;
    const bool split = g.acc != nullptr && (ihi - ilo) > g.chunk;

    uint64_t acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0;
    uint32_t since = 0;
    const int base = ORIGIN + int(threadIdx.x) * R;
    const int tid = threadIdx.x;
    uint32_t wr[NW], vr[NV];
    auto fetch = [&](int64_t ic) {  // chunk [ic, ic + MUL_TI) into registers
        const int cnt = int(i_end - ic < MUL_TI ? i_end - ic : MUL_TI);
        const int64_t off = k0 - ic - ORIGIN;  // sv[x] = b[x + off]
#pragma unroll
        for (int k = 0; k < NW; ++k) {
            const int u = tid + k * MUL_T;
            wr[k] = (u < MUL_TI && u < cnt) ? a[ic + u] : 0u;
        }
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int x = tid + k * MUL_T;
            const int64_t j = x + off;
            vr[k] = (x < SV && j >= 0 && j < nb) ? b[j] : 0u;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int k = 0; k < NW; ++k)
            if (tid + k * MUL_T < MUL_TI) sw[buf][tid + k * MUL_T] = wr[k];
#pragma unroll
        for (int k = 0; k < NV; ++k)
            if (tid + k * MUL_T < SV) sv[buf][tid + k * MUL_T] = vr[k];
    };
    fetch(i_begin);
    store(0);
    __syncthreads();
    int buf = 0;
    for (int64_t ic = i_begin; ic < i_end; ic += MUL_TI) {
        const int cnt = int(i_end - ic < MUL_TI ? i_end - ic : MUL_TI);
        const bool more = ic + MUL_TI < i_end;
        if (more) fetch(ic + MUL_TI);  // in flight during the multiply
#if MUL_GROUPED
        if constexpr (R % 4 == 0)
            conv_accumulate_grouped<R>(acc, sw[buf], (cnt + R - 1) / R, sv[buf], base, since, g.F);
        else
#endif
            conv_accumulate<R>(acc, sw[buf], (cnt + R - 1) / R, sv[buf], base, since, g.F);
        if (more) store(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }

    uint32_t* __restrict__ f = g.f + inst * g.ldf;
    const int64_t fbase = inst * g.ldf - g.klo;  // FAN: word k at every g.fan.p[q][fbase + k]
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t k = k0 + int64_t(threadIdx.x) * R + r;
        if (k < nf) {
            const uint32_t v = reduce(acc[r], g.F);
            if (split)
                atomicAdd(g.acc + (k - g.klo), (unsigned long long)v);
            else
                if constexpr (FAN)
                    fan_store<true>(g.fan, fbase + k, v);
                else
                    f[k - g.klo] = v;
        }
    }
    if (!split) return;
    // the last item to finish this k-tile reduces it (threadfence reduction)
    __shared__ bool last;
#if MUL_ARRIVE == 1
    __threadfence();
#endif
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned items = unsigned((ihi - ilo + g.chunk - 1) / g.chunk);
#if MUL_ARRIVE == 1
        last = atomicAdd(g.arrived + blockIdx.y, 1u) == items - 1;
#else
        // release: this CTA's accumulator REDs (ordered before the barrier
        // above by every thread's cumulativity through bar.sync) happen
        // before the arrival; acquire: the last arriver sees every item's
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old)
                     : "l"(g.arrived + blockIdx.y) : "memory");
        last = old == items - 1;
#endif
    }
    __syncthreads();
    if (!last) return;
#if MUL_ARRIVE == 1
    __threadfence();
#endif
    for (int t = threadIdx.x; t < TK; t += MUL_T) {
        const int64_t k = k0 + t;
        if (k < nf) {
            const uint32_t v = reduce(__ldcg(g.acc + (k - g.klo)), g.F);
            if constexpr (FAN)
                fan_store<true>(g.fan, fbase + k, v);
            else
                f[k - g.klo] = v;
            __stcg(g.acc + (k - g.klo), 0ull);  // zero for the next call on this stream
        }
    }
    if (threadIdx.x == 0) g.arrived[blockIdx.y] = 0u;
}

namespace {

int pick_tile(int64_t s, const FieldParams& F) {
    int R = 1;
    for (int c : {2, 4, 8, 16})
        if (c <= s) R = c;
    while (R > 1 && uint32_t(R) > F.fold_terms) R /= 2;
    return R;
}

template <int R>
void launch_tile(const MulArgs& g, dim3 grid, cudaStream_t st) {
    if (g.fan.n > 1)
        mul_kernel<R, true><<<grid, MUL_T, 0, st>>>(g);
    else
        mul_kernel<R, false><<<grid, MUL_T, 0, st>>>(g);
    check_launch("mul_kernel", grid, dim3(MUL_T));
}

void dispatch(int R, const MulArgs& g, dim3 grid, cudaStream_t st) {
    switch (R) {
        case 16: launch_tile<16>(g, grid, st); break;
        case 8: launch_tile<8>(g, grid, st); break;
        case 4: launch_tile<4>(g, grid, st); break;
        case 2: launch_tile<2>(g, grid, st); break;
        default: launch_tile<1>(g, grid, st); break;
    }
}

}  // namespace

void launch_mul(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb,
                uint32_t* f, int64_t s, int64_t l, cudaStream_t st) {
    launch_mul_range(F, a, na, b, nb, 0, na + nb - 1, f, s, l, st);
}

// Outputs [klo, khi) of the product into f[0, khi - klo): the per-rank slice of
// an output-range-sharded product.
void launch_mul_range(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b,
                      int64_t nb, int64_t klo, int64_t khi, uint32_t* f, int64_t s, int64_t l,
                      cudaStream_t st) {
    launch_mul_range_fan(F, a, na, b, nb, klo, khi, fan_of(f), s, l, st);
}

void launch_mul_range_fan(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b,
                          int64_t nb, int64_t klo, int64_t khi, Fan f, int64_t s, int64_t /*l*/,
                          cudaStream_t st) {
    if (klo == 0 && khi == na + nb - 1 && tcmul_single_supported(na, nb, s)) {
        launch_tcmul_single(F, a, na, b, nb, f, st);  // integer tensor core (tcmul.cu)
        return;
    }
    if (s <= 0) s = 8;  // auto on the CUDA cores: the 8 x 8 register tile
    const int R = pick_tile(s, F);
    const int64_t TK = int64_t(MUL_T) * R;
    const int64_t nf = khi - klo;
    if (nf <= 0) return;
    const int64_t nkt = ceil_div(nf, TK);
    if (nkt > 65535) throw Error(ST_INVALID, "multiplication: product too long for plain kernel");
    // Total staged terms over all k-tiles; aim for ~8 items per SM.
    int64_t total = 0, longest = 0;
    for (int64_t kt = 0; kt < nkt; ++kt) {
        const int64_t k0 = klo + kt * TK;
        const int64_t lo = std::max<int64_t>(0, k0 - (nb - 1)), hi = std::min<int64_t>(na, k0 + TK);
        total += hi - lo;
        longest = std::max(longest, hi - lo);
    }
    const int64_t target = 16LL * sm_count();
    int64_t chunk = ceil_div(ceil_div(total, target), MUL_TI) * MUL_TI;
    if (chunk < MUL_TI) chunk = MUL_TI;
    const int64_t items = ceil_div(longest, chunk);

    MulArgs g{};
    g.a = a;
    g.b = b;
    g.f = f.p[0];
    g.fan = f;
    g.na = na;
    g.nb = nb;
    g.chunk = chunk;
    g.klo = klo;
    g.khi = khi;
    g.F = F;
    if (items > 1) {  // the thread's all-zero accumulator and counters (ZeroBuf)
        const size_t words = size_t(nf) + size_t(ceil_div(nkt, 2));
        g.acc = zero_buf_acquire(words, st);
        g.arrived = reinterpret_cast<unsigned*>(g.acc + nf);
        dispatch(R, g, dim3(unsigned(items), unsigned(nkt), 1), st);
        zero_buf_release(st);
        return;
    }
    dispatch(R, g, dim3(unsigned(items), unsigned(nkt), 1), st);
}

void launch_mul_batched(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                        const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, uint32_t* Fo,
                        int64_t ldf, int64_t s, cudaStream_t st) {
    launch_mul_batched_fan(F, A, lda, na, B, ldb, nb, count, fan_of(Fo), ldf, s, st);
}

void launch_mul_batched_fan(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                            const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, Fan Fo,
                            int64_t ldf, int64_t s, cudaStream_t st) {
    if (tcmul_supported(na, nb, count, s)) {  // integer tensor core (tcmul.cu)
        launch_tcmul_batched(F, A, lda, na, B, ldb, nb, count, Fo, ldf, st);
        return;
    }
    if (s <= 0) s = 8;  // auto on the CUDA cores
    const int R = pick_tile(s, F);
    const int64_t TK = int64_t(MUL_T) * R;
    const int64_t nf = na + nb - 1;
    const int64_t nkt = ceil_div(nf, TK);
    if (nkt > 65535) throw Error(ST_INVALID, "multiplication: product too long for plain kernel");
    MulArgs g{};
    g.na = na;
    g.nb = nb;
    g.lda = lda;
    g.ldb = ldb;
    g.ldf = ldf;
    g.chunk = na + nb;  // one item per k-tile: no split, direct stores
    g.klo = 0;
    g.khi = nf;
    g.F = F;
    for (int64_t c0 = 0; c0 < count; c0 += 65535) {
        const int64_t c = std::min<int64_t>(65535, count - c0);
        g.a = A + c0 * lda;
        g.b = B + c0 * ldb;
        g.fan = fan_offset(Fo, c0 * ldf);
        g.f = g.fan.p[0];
        dispatch(R, g, dim3(1, unsigned(nkt), unsigned(c)), st);
    }
}

}  // namespace mmm_cu
