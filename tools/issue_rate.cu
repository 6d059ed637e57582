// issue_rate.cu -- single-warp issue rate of IMAD, IMAD.HI and IMAD.WIDE
// (8 independent chains per thread, so latency is hidden), cycles per warp
// instruction; and with 4 warps on one SM (one per SMSP).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/issue_rate tools/issue_rate.cu
#include <cstdio>
#include <cstdint>
template <int K>
__global__ void k(const uint32_t* in, long long* out, uint32_t* sink, int iters) {
    uint32_t a[8], b = in[threadIdx.x & 7] | 1u;
    uint64_t w[8];
    for (int i = 0; i < 8; ++i) { a[i] = in[i + threadIdx.x] | 1u; w[i] = a[i]; }
    __syncwarp();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (K == 0) a[i] = a[i] * b + 7u;                           // IMAD
            if (K == 1) a[i] = __umulhi(a[i], b) + a[i];                  // IMAD.HI (+IADD)
            if (K == 2) w[i] = w[i] + uint64_t(uint32_t(w[i] >> 7)) * b; // IMAD.WIDE acc
            if (K == 3) w[i] = uint64_t(a[i]) * b + w[i], a[i] ^= uint32_t(w[i]);  // WIDE + LOP
        }
    }
    __syncwarp();
    const long long t = clock64() - t0;
    if (threadIdx.x == 0) out[blockIdx.x] = t;
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s ^= a[i] ^ uint32_t(w[i]) ^ uint32_t(w[i] >> 32);
    sink[threadIdx.x] = s;
}
int main() {
    uint32_t *in, *sink; long long* out;
    cudaMallocManaged(&in, 4096); cudaMallocManaged(&out, 64); cudaMalloc(&sink, 4096);
    for (int i = 0; i < 1024; ++i) in[i] = 2654435761u * i;
    const int it = 10000;
    const char* nm[] = {"imad", "imad_hi", "imad_wide_acc", "wide_plus_lop"};
    for (int warps : {1, 4}) {
        for (int K = 0; K < 4; ++K) {
            for (int r = 0; r < 2; ++r) {
                if (K == 0) k<0><<<1, 32 * warps>>>(in, out, sink, it);
                if (K == 1) k<1><<<1, 32 * warps>>>(in, out, sink, it);
                if (K == 2) k<2><<<1, 32 * warps>>>(in, out, sink, it);
                if (K == 3) k<3><<<1, 32 * warps>>>(in, out, sink, it);
                cudaDeviceSynchronize();
            }
            printf("warps=%d %s: %.2f cycles per warp-instruction-group (8 chains)\n", warps, nm[K], out[0] / (8.0 * it));
        }
    }
    return 0;
}
