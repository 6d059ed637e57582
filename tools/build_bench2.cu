// build_bench2.cu -- cycles of the head's window build (build_window_part,
// BUILD_PARTS warps) in isolation, cold and warm, from clock64 on warp 0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/build_bench2 tools/build_bench2.cu
#include <cstdlib>
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

__global__ void kern(const uint32_t* rnd, long long* out, uint32_t* sink, FieldParams F, int warps) {
    __shared__ __align__(16) uint32_t Ps[4 * PL], topA[W1 + PL + 4], topB[W1 + PL + 4],
        red[BUILD_PARTS * 2 * W1];
    __shared__ int hi[4];
    for (int i = threadIdx.x; i < 4 * PL; i += blockDim.x) Ps[i] = rnd[i] % F.p;
    for (int i = threadIdx.x; i < W1 + PL + 4; i += blockDim.x) {
        topA[i] = rnd[512 + i] % F.p;
        topB[i] = rnd[1024 + i] % F.p;
    }
    if (threadIdx.x < 4) hi[threadIdx.x] = PL - 1;
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    long long t[4];
    for (int rep = 0; rep < 4; ++rep) {
        __syncthreads();
        const long long t0 = clock64();
        if (warp < warps) build_window_part(warp, red, Ps, hi, topA, topB, F);
        __syncwarp();
        t[rep] = clock64() - t0;
    }
    if (threadIdx.x == 0)
        for (int i = 0; i < 4; ++i) out[i] = t[i];
    __syncthreads();
    sink[threadIdx.x] = red[threadIdx.x];
}

int main() {
    const FieldParams F = make_field(469762049u);
    uint32_t *rnd, *sink;
    long long* out;
    cudaMallocManaged(&rnd, 4096 * 4);
    cudaMallocManaged(&out, 64);
    cudaMalloc(&sink, 4096);
    for (int i = 0; i < 4096; ++i) rnd[i] = uint32_t(i * 2654435761u);
    for (int w : {1, BUILD_PARTS}) {
        kern<<<1, 256>>>(rnd, out, sink, F, w);
        cudaDeviceSynchronize();
        printf("warps=%d build cycles (warp 0): %lld %lld %lld %lld\n", w, out[0], out[1], out[2], out[3]);
    }
    return 0;
}
