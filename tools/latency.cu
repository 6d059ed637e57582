// latency.cu -- dependent-chain latencies (cycles) of the instructions on the
// GCD chain's critical path, one warp, clock64 around N dependent ops.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/latency tools/latency.cu
#include <cstdint>
#include <cstdio>

constexpr int N = 4096;

__global__ void k(const uint32_t* in, long long* out, uint32_t* sink) {
    __shared__ uint32_t sm[64];
    const int lane = threadIdx.x & 31;
    uint32_t a = in[lane], b = in[lane + 32] | 1u, p = 469762049u, pinv = in[2] | 1u;
    sm[lane] = a;
    sm[lane + 32] = b;
    __syncwarp();
    long long t0, t1;
    // 1) SHFL.IDX dependent chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) a = __shfl_sync(0xffffffffu, a, (a + lane) & 31);
    t1 = clock64();
    out[0] = t1 - t0;
    // 2) IMAD.WIDE.U32 accumulate chain
    uint64_t acc = a;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) acc = uint64_t(uint32_t(acc)) * b + acc;
    t1 = clock64();
    out[1] = t1 - t0;
    // 3) lazy REDC comb chain: y*a + nx*b -> m -> hi - mp + p
    uint32_t x = a ^ uint32_t(acc), y = b;
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) {
        const uint64_t t = uint64_t(y) * x + uint64_t(2 * p - y) * b;
        const uint32_t m = uint32_t(t) * pinv;
        x = uint32_t(t >> 32) - __umulhi(m, p) + p;
    }
    t1 = clock64();
    out[2] = t1 - t0;
    // 4) VOTE.ANY (ballot) chain
    uint32_t v = x;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) v = __ballot_sync(0xffffffffu, (v >> (lane & 7)) & 1) + lane;
    t1 = clock64();
    out[3] = t1 - t0;
    // 5) LDS dependent chain
    uint32_t idx = v & 63;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) idx = sm[idx & 63];
    t1 = clock64();
    out[4] = t1 - t0;
    // 6) shuffle-broadcast + compare + branch (the fast-path "h1" pattern)
    uint32_t h = idx;
    int cnt = 0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        h = __shfl_sync(0xffffffffu, h + 1, 1);
        if (h != 0u && h != p) ++cnt;
    }
    t1 = clock64();
    out[5] = t1 - t0;
    // 7) 6 independent SHFLs per iteration, then one combining op (throughput)
    uint32_t q0 = h, q1 = h ^ 1u, q2 = h ^ 2u, q3 = h ^ 3u, q4 = h ^ 4u, q5 = h ^ 5u;
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        q0 = __shfl_sync(0xffffffffu, q0, (lane + 1) & 31);
        q1 = __shfl_sync(0xffffffffu, q1, (lane + 2) & 31);
        q2 = __shfl_sync(0xffffffffu, q2, (lane + 3) & 31);
        q3 = __shfl_sync(0xffffffffu, q3, (lane + 4) & 31);
        q4 = __shfl_sync(0xffffffffu, q4, (lane + 5) & 31);
        q5 = __shfl_sync(0xffffffffu, q5, (lane + 6) & 31);
        q0 ^= q5;
    }
    t1 = clock64();
    out[6] = t1 - t0;
    // 8) IMAD.HI dependent chain
    uint32_t hh = q0 | 1u;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) hh = __umulhi(hh, b) + lane;
    t1 = clock64();
    out[7] = t1 - t0;
    // 9) Shoup product chain: q = hi(a' x); x = a x - q p
    uint32_t sx = hh, sa = b % p, sq = 0x5a5a5a5au;
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) {
        const uint32_t qq = __umulhi(sq, sx);
        sx = sa * sx - qq * p;
    }
    t1 = clock64();
    out[8] = t1 - t0;
    // 10) comb3 chain (3 IMAD.WIDE accumulate + REDC)
    uint32_t cx = sx;
    t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) {
        const uint64_t t = uint64_t(y) * cx + uint64_t(b) * (cx ^ 7u) + uint64_t(sa) * (cx + 3u);
        const uint32_t m = uint32_t(t) * pinv;
        cx = uint32_t(t >> 32) - __umulhi(m, p) + p;
    }
    t1 = clock64();
    out[9] = t1 - t0;
    // 11) rolled loop of one dependent IADD (back-edge cost)
    uint32_t lx = cx;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) lx = lx * 3u + 1u;
    t1 = clock64();
    out[10] = t1 - t0;
    // 12) rolled loop with a data-dependent uniform if/else (both sides used)
    uint32_t bx = lx;
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        const uint32_t u = __shfl_sync(0xffffffffu, bx, 0);
        if (u & 1u) bx = bx * 3u + 1u;
        else bx = (bx >> 1) ^ 0x1234u;
    }
    t1 = clock64();
    out[11] = t1 - t0;
    sink[threadIdx.x] = a + uint32_t(acc) + x + v + idx + h + cnt + q0 + q1 + q2 + q3 + q4 + hh + sx + cx + lx + bx;
}

int main() {
    uint32_t* in;
    long long* out;
    uint32_t* sink;
    cudaMallocManaged(&in, 256);
    cudaMallocManaged(&out, 128);
    cudaMalloc(&sink, 128);
    for (int i = 0; i < 64; ++i) in[i] = 0x9e3779b9u * (i + 1);
    k<<<1, 32>>>(in, out, sink);
    cudaDeviceSynchronize();
    k<<<1, 32>>>(in, out, sink);
    cudaDeviceSynchronize();
    const char* names[] = {"shfl_idx", "imad_wide_acc", "lazy_redc_comb", "vote_ballot", "lds", "shfl_bcast_cmp_branch", "shfl6_indep_iter", "imad_hi", "shoup_chain", "comb3_chain", "rolled_loop_imad", "rolled_loop_bcast_ifelse"};
    printf("{");
    for (int i = 0; i < 12; ++i) printf("%s\"%s\": %.2f", i ? ", " : "", names[i], double(out[i]) / N);
    printf("}\n");
    return 0;
}
