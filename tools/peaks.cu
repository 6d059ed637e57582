// peaks.cu -- integer-pipe microbenchmarks for the roofline denominators
// (SURVEY.md §7 step 1).  Sustained rate of IMAD.WIDE.U32 with a 64-bit
// addend (one lazy modular MAD) in several operand patterns -- the best one
// is the "modular-MAD peak" -- plus IMAD and IMAD.HI.  Every SM busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
// Prints one JSON object.
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

constexpr int ITERS = 2048;

// P1: 16 independent chains acc += lo(acc) * b
__global__ void k_wide_chain(const uint32_t* in, uint64_t* out) {
    constexpr int CH = 16;
    const uint32_t b = in[threadIdx.x & 31] | 1u;
    uint64_t acc[CH];
    for (int c = 0; c < CH; ++c) acc[c] = in[(threadIdx.x + c) & 63];
#pragma unroll 2
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] += uint64_t(uint32_t(acc[c])) * b;
    uint64_t s = 0;
    for (int c = 0; c < CH; ++c) s ^= acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// P2: the 8x8 register tile of the product kernel: acc[r] += X[t] * W[7 + r - t],
// operands refreshed by cheap ALU ops so nothing is loop-invariant.
__global__ void k_wide_tile(const uint32_t* in, uint64_t* out) {
    constexpr int R = 8;
    uint32_t X[R], W[2 * R - 1];
    uint64_t acc[R];
    for (int j = 0; j < R; ++j) {
        X[j] = in[(threadIdx.x + j) & 63];
        acc[j] = j;
    }
    for (int j = 0; j < 2 * R - 1; ++j) W[j] = in[(threadIdx.x + 3 * j) & 63];
    for (int i = 0; i < ITERS / 8; ++i) {
#pragma unroll
        for (int t = 0; t < R; ++t)
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] += uint64_t(X[t]) * W[(R - 1) + r - t];
#pragma unroll
        for (int j = 0; j < R; ++j) X[j] = X[j] * 0x9e3779b9u + 1u;  // keep operands live
    }
    uint64_t s = 0;
    for (int r = 0; r < R; ++r) s ^= acc[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_lo(const uint32_t* in, uint64_t* out) {
    constexpr int CH = 16;
    uint32_t a[CH], b = in[threadIdx.x & 31] | 1u, acc[CH];
    for (int c = 0; c < CH; ++c) {
        a[c] = in[(threadIdx.x + c) & 63];
        acc[c] = c;
    }
#pragma unroll 2
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] = acc[c] * b + a[c];  // IMAD
    uint64_t s = 0;
    for (int c = 0; c < CH; ++c) s ^= acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_hi(const uint32_t* in, uint64_t* out) {
    constexpr int CH = 16;
    uint32_t a[CH], b = in[threadIdx.x & 31] | 1u;
    for (int c = 0; c < CH; ++c) a[c] = in[(threadIdx.x + c) & 63] | 0x80000000u;
#pragma unroll 2
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = __umulhi(a[c], b) ^ a[c];  // IMAD.HI + LOP3
    uint64_t s = 0;
    for (int c = 0; c < CH; ++c) s ^= a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K>
double best_seconds(K k, int blocks, int threads, const uint32_t* in, uint64_t* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<blocks, threads>>>(in, out);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 7; ++r) {
        cudaEventRecord(e0);
        k<<<blocks, threads>>>(in, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best * 1e-3;
}

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int threads = 256, blocks = sms * 8;
    uint32_t* in;
    uint64_t* out;
    cudaMalloc(&in, 256);
    cudaMemset(in, 0x5b, 256);
    cudaMalloc(&out, size_t(blocks) * threads * 8);
    const double n = double(blocks) * threads;
    const double chain = n * ITERS * 16 / best_seconds(k_wide_chain, blocks, threads, in, out);
    const double tile = n * (ITERS / 8) * 64 / best_seconds(k_wide_tile, blocks, threads, in, out);
    const double lo = n * ITERS * 16 / best_seconds(k_lo, blocks, threads, in, out);
    const double hi = n * ITERS * 16 / best_seconds(k_hi, blocks, threads, in, out);
    const double best = chain > tile ? chain : tile;
    printf("{\"sms\": %d, \"imad_wide_per_s\": %.4e, \"imad_wide_chain_per_s\": %.4e, "
           "\"imad_wide_tile8x8_per_s\": %.4e, \"imad_per_s\": %.4e, \"imad_hi_per_s\": %.4e}\n",
           sms, best, chain, tile, lo, hi);
    return 0;
}
