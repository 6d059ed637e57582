// poll_lat.cu -- store-to-poller visibility latency on this GPU: CTA 0 writes a
// tagged 64-bit word (st.relaxed.gpu) every `gap` ns; CTAs 1..G-1 (one warp
// each) poll it with ld.relaxed.gpu and record %globaltimer when they see each
// tag.  Prints the mean delay publish -> seen, for 1 and for all pollers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/poll_lat tools/poll_lat.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ long long gt() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint64_t ld64(const uint64_t* p) { uint64_t v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p)); return v; }
__device__ __forceinline__ void st64(uint64_t* p, uint64_t v) { asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory"); }

__global__ void k(uint64_t* word, long long* tpub, long long* sum, int iters, int npoll, int mode) {
    if (blockIdx.x == 0) {
        if (threadIdx.x != 0) return;
        for (int i = 1; i <= iters; ++i) {
            const long long t0 = gt();
            while (gt() - t0 < 4000) {}
            const long long t = gt();
            tpub[i] = t;
            if (mode == 1) __threadfence();  // make tpub visible first (only for the check)
            st64(word, (uint64_t(i) << 32) | 7u);
        }
        return;
    }
    if (int(blockIdx.x) > npoll || threadIdx.x >= 32) return;
    long long acc = 0;
    for (int i = 1; i <= iters; ++i) {
        uint64_t w = ld64(word);
        while (!__all_sync(0xffffffffu, unsigned(w >> 32) >= unsigned(i))) w = ld64(word);
        const long long t = gt();
        if (threadIdx.x == 0) acc += t;
    }
    if (threadIdx.x == 0) atomicAdd((unsigned long long*)sum, (unsigned long long)acc);
}
int main() {
    uint64_t* w; long long *tp, *sum;
    cudaMalloc(&w, 8); cudaMallocManaged(&tp, 8 * 1001); cudaMallocManaged(&sum, 8);
    const int it = 1000;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int np : {1, 8, sms - 1}) {
        cudaMemset(w, 0, 8); *sum = 0; cudaDeviceSynchronize();
        k<<<sms, 32>>>(w, tp, sum, it, np, 0);
        cudaDeviceSynchronize();
        long long tsum = 0; for (int i = 1; i <= it; ++i) tsum += tp[i];
        printf("pollers=%d mean publish->seen %.1f ns\n", np, double(*sum - tsum * np) / (double(it) * np));
    }
    return 0;
}
