// replay_bench.cu -- one warp, dependent iterations of the replay's fused
// entry (three shifted copies + 3-term Montgomery reduction per word) and its
// parts, to find which one sets the per-entry latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/replay_bench tools/replay_bench.cu
#include <cstdint>
#include <cstdio>

constexpr int PE = 2, N = 4096;

template <int K>
__device__ __forceinline__ void shr(const uint32_t (&w)[PE], uint32_t (&o)[PE]) {
    const int lane = threadIdx.x & 31;
    uint32_t r[PE];
#pragma unroll
    for (int e = 0; e < PE; ++e) r[e] = __shfl_sync(0xffffffffu, w[e], (lane - K) & 31);
#pragma unroll
    for (int e = 0; e < PE; ++e) o[e] = lane < K ? (e > 0 ? r[e - 1] : 0u) : r[e];
}
__device__ __forceinline__ uint32_t comb3(uint32_t a, uint32_t x, uint32_t b, uint32_t y, uint32_t c,
                                          uint32_t z, uint32_t p, uint32_t pinv) {
    const uint64_t t = uint64_t(a) * x + uint64_t(b) * y + uint64_t(c) * z;
    const uint32_t m = uint32_t(t) * pinv;
    return uint32_t(t >> 32) - __umulhi(m, p) + p;
}

template <int V>
__global__ void k(const uint32_t* in, uint32_t* out, long long* cyc, uint32_t p, uint32_t pinv) {
    const int lane = threadIdx.x;
    uint32_t u[PE], v[PE];
    for (int e = 0; e < PE; ++e) {
        u[e] = in[e * 32 + lane];
        v[e] = in[64 + e * 32 + lane];
    }
    const uint32_t a = in[200], b = in[201], c = in[202];
    const long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) {
        uint32_t us2[PE], vs2[PE], vs1[PE];
        if (V == 1) {  // no shuffles
            for (int e = 0; e < PE; ++e) us2[e] = u[e], vs2[e] = v[e], vs1[e] = v[e] ^ 1u;
        } else {
            shr<2>(u, us2);
            shr<2>(v, vs2);
            shr<1>(v, vs1);
        }
        uint32_t n[PE];
#pragma unroll
        for (int e = 0; e < PE; ++e) {
            if (V == 2) n[e] = us2[e] ^ vs2[e] ^ vs1[e];  // no arithmetic
            else n[e] = comb3(a, us2[e], b, vs2[e], c, vs1[e], p, pinv);
        }
        // roles alternate: the new row is the next divisor
#pragma unroll
        for (int e = 0; e < PE; ++e) {
            u[e] = v[e];
            v[e] = n[e];
        }
    }
    __syncwarp();
    const long long t = clock64() - t0;
    for (int e = 0; e < PE; ++e) out[e * 32 + lane] = u[e] ^ v[e];
    if (lane == 0) cyc[V] = t;
}

int main() {
    uint32_t *in, *out;
    long long* cyc;
    cudaMallocManaged(&in, 1024 * 4);
    cudaMallocManaged(&out, 1024 * 4);
    cudaMallocManaged(&cyc, 64);
    for (int i = 0; i < 1024; ++i) in[i] = (i * 2654435761u) % 469762049u;
    const uint32_t p = 469762049u;
    uint32_t pinv = 1;
    for (int i = 0; i < 5; ++i) pinv *= 2 - p * pinv;
    pinv = 0u - pinv;  // -p^-1 mod 2^32 ... sign irrelevant for timing
    for (int rep = 0; rep < 2; ++rep) {
        k<0><<<1, 32>>>(in, out, cyc, p, pinv);
        k<1><<<1, 32>>>(in, out, cyc, p, pinv);
        k<2><<<1, 32>>>(in, out, cyc, p, pinv);
        cudaDeviceSynchronize();
    }
    printf("{\"full\": %.1f, \"no_shfl\": %.1f, \"shfl_only\": %.1f}\n", double(cyc[0]) / N,
           double(cyc[1]) / N, double(cyc[2]) / N);
    return 0;
}
