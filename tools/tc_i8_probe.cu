// tc_i8_probe.cu -- measurement-only probe of the sm_100a integer tensor core
// (tcgen05.mma kind::i8, u8 x u8 -> s32 in TMEM) for the limb-split exact
// product:
//   1. correctness of the descriptors/layouts in csrc/tc.cuh: one 128 x N x 128
//      UMMA product against a CPU reference (exact int32);
//   2. throughput: every SM issues back-to-back 128 x N x 32 MMAs from shared
//      memory; MAC/s over the grid (CUDA events) vs 148 x 8192 MAC/clk.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_1402_0264_b200/csrc tools/tc_i8_probe.cu -o tools/tc_i8_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc.cuh"

using namespace mmm_cu;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

__device__ int g_shift = 0, g_bo = 0;

template <int N>
__global__ void __launch_bounds__(128) probe_kernel(const uint8_t* A, const uint8_t* B, int32_t* D,
                                                    int iters, int col_off) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = sm;              // 128 x 128 B
    uint8_t* sB = sm + 128 * 128;  // N x 128 B
    __shared__ uint64_t mbar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * 128; i += 128) sA[tc::sw128(i >> 7, i & 127)] = A[i];
    const int shift = g_shift;
    for (int i = tid; i < (N + 8) * 128; i += 128) sB[i] = 0;
    __syncthreads();
    for (int i = tid; i < N * 128; i += 128) sB[tc::sw128((i >> 7) + shift, i & 127)] = B[i];
    tc::fence_async_smem();
    if (warp == 0) tc::tmem_alloc<512>(&tslot);
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tbase = tslot;
    constexpr uint32_t idesc = tc::idesc_u8(128, N);
    if (tid == 0) {
        const uint32_t a0 = tc::smem_u32(sA), b0 = tc::smem_u32(sB);
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                tc::mma_u8(tbase + col_off, tc::desc_sw128(a0 + 32 * k),
                           tc::desc_sw128(b0 + 128 * shift + 32 * k) | (uint64_t(g_bo & 7) << 49), idesc,
                           (it | k) != 0);
        tc::commit(&mbar);
    }
    __syncwarp();
    tc::mbar_wait(&mbar, 0);
    tc::fence_after_sync();
    if (D) {
        const int row = warp * 32 + (tid & 31);
        // aligned reads of columns [c0, c0 + 32) covering [col_off, col_off + N)
        for (int c0 = 0; c0 < N + col_off; c0 += 32) {
            uint32_t v[32];
            tc::tmem_ld32(tbase + (uint32_t(warp * 32) << 16) + c0, v);
            tc::tmem_ld_wait();
            for (int j = 0; j < 32; ++j) {
                const int col = c0 + j - col_off;
                if (col >= 0 && col < N) D[(size_t(blockIdx.x) * 128 + row) * N + col] = int32_t(v[j]);
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tbase);
}

template <int N>
void run(int sms, int col_off = 0) {
    const size_t smem = 1024 + 128 * 128 + (N + 8) * 128;
    CK(cudaFuncSetAttribute(probe_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    std::vector<uint8_t> A(128 * 128), B(N * 128);
    srand(7 + N);
    for (auto& x : A) x = uint8_t(rand());
    for (auto& x : B) x = uint8_t(rand());
    uint8_t *dA, *dB;
    int32_t* dD;
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, B.size()));
    CK(cudaMalloc(&dD, size_t(128) * N * 4));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
    probe_kernel<N><<<1, 128, smem>>>(dA, dB, dD, 1, col_off);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> D(size_t(128) * N);
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int i = 0; i < 128; ++i)
        for (int j = 0; j < N; ++j) {
            int32_t s = 0;
            for (int k = 0; k < 128; ++k) s += int32_t(A[i * 128 + k]) * int32_t(B[j * 128 + k]);
            if (s != D[size_t(i) * N + j]) {
                if (bad < 5) printf("  mismatch N=%d D[%d][%d]=%d want %d\n", N, i, j, D[size_t(i) * N + j], s);
                ++bad;
            }
        }
    printf("correctness N=%d col_off=%d: %s (%ld bad of %d)\n", N, col_off, bad ? "FAIL" : "ok", bad, 128 * N);
    if (col_off) return;
    // throughput: one CTA per SM, `iters` x 4 MMAs of 128 x N x 32
    const int iters = 4096;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    probe_kernel<N><<<sms, 128, smem>>>(dA, dB, nullptr, 64, 0);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(e0));
        probe_kernel<N><<<sms, 128, smem>>>(dA, dB, nullptr, iters, 0);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    const double macs = double(sms) * iters * 4 * 128.0 * N * 32;
    printf("throughput N=%d: %.3f ms, %.3e MAC/s (%.1f%% of 148 x 8192 MAC/clk at 1965 MHz)\n", N,
           best, macs / (best * 1e-3), 100.0 * macs / (best * 1e-3) / (148.0 * 8192 * 1.965e9));
    CK(cudaFree(dA));
    CK(cudaFree(dB));
    CK(cudaFree(dD));
}

int main(int argc, char** argv) {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    if (argc > 2) {  // B operand starting `shift` rows into its swizzle atom, base_offset bo
        int sh = atoi(argv[1]), bo = atoi(argv[2]);
        CK(cudaMemcpyToSymbol(g_shift, &sh, sizeof(int)));
        CK(cudaMemcpyToSymbol(g_bo, &bo, sizeof(int)));
        printf("shift=%d bo=%d: ", sh, bo);
        run<224>(sms, 2);
        return 0;
    }
    if (argc > 1) {  // one correctness case at a column offset
        run<224>(sms, atoi(argv[1]));
        return 0;
    }
    run<32>(sms);
    run<64>(sms);
    run<128>(sms);
    run<256>(sms);
    run<224>(sms);
    return 0;
}
