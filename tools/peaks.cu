// peaks.cu -- integer-pipe microbenchmarks for the roofline denominators
// (SURVEY.md §7 step 1): sustained issue rate of IMAD.WIDE.U32 with a 64-bit
// addend (one lazy modular MAD), IMAD (32-bit), IMAD.HI.U32, and the SM clock
// under that load.  Many independent chains per thread, every SM busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
// Prints one JSON object.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 16;      // independent chains per thread
constexpr int ITERS = 4096;

__global__ void k_wide(const uint32_t* in, uint64_t* out, long long* clk) {
    uint32_t a[CH], b = in[threadIdx.x & 31] | 1u;
    uint64_t acc[CH];
    for (int c = 0; c < CH; ++c) { a[c] = in[(threadIdx.x + c) & 63]; acc[c] = c; }
    long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] += uint64_t(uint32_t(acc[c])) * b;  // IMAD.WIDE.U32
    long long t1 = clock64();
    uint64_t s = 0;
    for (int c = 0; c < CH; ++c) s ^= acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

__global__ void k_lo(const uint32_t* in, uint32_t* out) {
    uint32_t a[CH], b = in[threadIdx.x & 31] | 1u, acc[CH];
    for (int c = 0; c < CH; ++c) { a[c] = in[(threadIdx.x + c) & 63]; acc[c] = c; }
#pragma unroll 4
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] = acc[c] * b + a[c];  // IMAD
    uint32_t s = 0;
    for (int c = 0; c < CH; ++c) s ^= acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_hi(const uint32_t* in, uint32_t* out) {
    uint32_t a[CH], b = in[threadIdx.x & 31] | 1u;
    for (int c = 0; c < CH; ++c) a[c] = in[(threadIdx.x + c) & 63] | 0x80000000u;
#pragma unroll 4
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = __umulhi(a[c], b) ^ a[c];  // IMAD.HI + LOP
    uint32_t s = 0;
    for (int c = 0; c < CH; ++c) s ^= a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K, class... A>
double time_kernel(K k, int blocks, int threads, A... args) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<<<blocks, threads>>>(args...);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k<<<blocks, threads>>>(args...);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best * 1e-3;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const int threads = 512, blocks = sms * 4;
    uint32_t* in;
    uint64_t* out64;
    uint32_t* out32;
    long long* clk;
    cudaMalloc(&in, 256);
    cudaMemset(in, 0x5b, 256);
    cudaMalloc(&out64, size_t(blocks) * threads * 8);
    cudaMalloc(&out32, size_t(blocks) * threads * 4);
    cudaMalloc(&clk, blocks * 8);
    const double ops = double(blocks) * threads * ITERS * CH;
    double t_wide = time_kernel(k_wide, blocks, threads, (const uint32_t*)in, out64, clk);
    long long c0;
    cudaMemcpy(&c0, clk, 8, cudaMemcpyDeviceToHost);
    double t_lo = time_kernel(k_lo, blocks, threads, (const uint32_t*)in, out32);
    double t_hi = time_kernel(k_hi, blocks, threads, (const uint32_t*)in, out32);
    // cycles of one block's loop vs its wall time -> effective SM clock
    const double per_sm_wide = ops / sms / (double)c0;
    printf("{\"sms\": %d, \"imad_wide_per_s\": %.4e, \"imad_per_s\": %.4e, \"imad_hi_per_s\": %.4e, "
           "\"imad_wide_per_clk_per_sm_est\": %.2f, \"block_cycles\": %lld, \"t_wide_s\": %.6f, "
           "\"clock_rate_attr_mhz\": %.0f}\n",
           sms, ops / t_wide, ops / t_lo, ops / t_hi, per_sm_wide, c0, t_wide,
           clk_khz / 1e3);
    return 0;
}
