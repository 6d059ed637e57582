// build_bench.cu -- cycles of the GCD window builder (build_window_part in
// paper_1402_0264_b200/csrc/gcd.cu) on synthetic P and top regions, run as in
// the head CTA (warps 0-6, warp 0 taking the last 32 items), and all 8 warps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/build_bench tools/build_bench.cu
#include "../paper_1402_0264_b200/csrc/gcd.cu"

namespace mmm_cu {
std::atomic<uint64_t> g_launches{0};
Arena& arena_for(cudaStream_t) {
    static Arena a;
    return a;
}
Scratch::Scratch(cudaStream_t s) : stream(s), arena(&arena_for(s)), ci0(0), off0(0) {}
void* Scratch::get_bytes(size_t b) {
    void* p = nullptr;
    cudaMalloc(&p, b);
    return p;
}
Scratch::~Scratch() {}
}  // namespace mmm_cu

using namespace mmm_cu;

__global__ void bench(const uint32_t* rnd, long long* out, uint32_t* sink, int reps, FieldParams F) {
    __shared__ __align__(16) uint32_t win[2 * W1], top[2 * (W1 + PL)], Ps[4 * PL],
        red[BUILD_PARTS * 2 * W1];
    __shared__ int hi[4];
    for (int i = threadIdx.x; i < 2 * (W1 + PL); i += blockDim.x) top[i] = rnd[i] % F.p;
    for (int i = threadIdx.x; i < 4 * PL; i += blockDim.x) Ps[i] = rnd[1024 + i] % F.p;
    if (threadIdx.x < 4) hi[threadIdx.x] = PL - 2;
    __syncthreads();
    long long c7 = 0, c8 = 0;
    for (int r = 0; r < reps; ++r) {
        __syncthreads();
        long long t0 = clock64();
        if (threadIdx.x < BUILDERS) {
            if ((threadIdx.x >> 5) < BUILD_PARTS)
                build_window_part(threadIdx.x >> 5, red, Ps, hi, top, top + W1 + PL, F);
            bar_sync(2, BUILDERS);
            if (threadIdx.x < 2 * W1) {
                uint64_t sum = 0;
                for (int pt = 0; pt < BUILD_PARTS; ++pt) sum += red[pt * 2 * W1 + threadIdx.x];
                win[threadIdx.x] = reduce(sum, F);
            }
            bar_sync(2, BUILDERS);
        }
        if (threadIdx.x == 0) c7 += clock64() - t0;
        __syncthreads();
        t0 = clock64();
        if ((threadIdx.x >> 5) < BUILD_PARTS)
            build_window_part(threadIdx.x >> 5, red, Ps, hi, top, top + W1 + PL, F);
        __syncthreads();
        if (threadIdx.x == 0) c8 += clock64() - t0;
    }
    if (threadIdx.x == 0) {
        out[0] = c7 / reps;
        out[1] = c8 / reps;
    }
    sink[threadIdx.x] = win[threadIdx.x & (2 * W1 - 1)];
}

int main() {
    const FieldParams F = make_field(469762049u);
    uint32_t *rnd, *sink;
    long long* out;
    cudaMallocManaged(&rnd, 4096 * 4);
    cudaMallocManaged(&out, 64);
    cudaMalloc(&sink, 1024 * 4);
    for (int i = 0; i < 4096; ++i) rnd[i] = uint32_t(i * 2654435761u);
    bench<<<1, GCD_T>>>(rnd, out, sink, 10, F);
    cudaDeviceSynchronize();
    bench<<<1, GCD_T>>>(rnd, out, sink, 100, F);
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"builder_7warps\": %lld, \"builder_8warps\": %lld, \"err\": \"%s\"}\n", out[0], out[1],
           cudaGetErrorString(e));
    return 0;
}
