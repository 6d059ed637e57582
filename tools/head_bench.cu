// head_bench.cu -- the division pipeline's head CTA (pipe_head in
// paper_1402_0264_b200/csrc/divmod.cu) alone: one CTA, bulk progress faked as
// complete, synthetic dividend/divisor; prints the head's stats (cycles).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/head_bench tools/head_bench.cu
#include "../paper_1402_0264_b200/csrc/divmod.cu"

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

__global__ void __launch_bounds__(PIPE_T, 1) head_only(PipeArgs g) {
    extern __shared__ __align__(16) uint32_t smem[];
    if (threadIdx.x < 32)
        inverse_series(g.h_glob, g.S, g.nb - 1,
                       [&](int64_t t) { return t <= g.nb - 1 ? g.b[g.nb - 1 - t] : 0u; }, g.F);
    __syncthreads();
    pipe_head_split(g, smem, 1);
}

int main(int argc, char** argv) {
    const int S = argc > 1 ? atoi(argv[1]) : 128;
    const int64_t na = 65537, nb = 32769;
    const FieldParams F = make_field(469762049u);
    uint32_t *a, *b, *q, *A, *h;
    unsigned* flags;
    long long* st;
    cudaMallocManaged(&a, na * 4);
    cudaMallocManaged(&b, nb * 4);
    cudaMalloc(&q, na * 4);
    cudaMallocManaged(&A, na * 4);
    cudaMalloc(&h, 4096 * 4);
    cudaMallocManaged(&flags, 64);
    cudaMallocManaged(&st, 16 * 8);
    uint64_t x = 88172645463325252ull;
    for (int64_t i = 0; i < na; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        a[i] = A[i] = uint32_t(x % 469762049u);
    }
    for (int64_t i = 0; i < nb; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        b[i] = uint32_t(x % 469762049u) | 1u;
    }
    flags[0] = 0;
    flags[1] = 1u << 30;  // progress of the single fake bulk owner: always ahead
    PipeArgs g{};
    g.a = a; g.b = b; g.q = q; g.r = nullptr; g.na = na; g.nb = nb; g.S = S; g.F = F;
    uint64_t* lam_t;
    cudaMalloc(&lam_t, size_t(na) * 8);
    g.A = A; g.h_glob = h; g.lam_t = lam_t; g.progress = flags + 1; g.stats = st;
    const size_t bytes = 64 * 1024;
    cudaFuncSetAttribute(head_only, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    for (int rep = 0; rep < 2; ++rep) {
        for (int i = 0; i < 16; ++i) st[i] = 0;
        head_only<<<1, PIPE_T, bytes>>>(g);
        cudaError_t e = cudaDeviceSynchronize();
        if (rep == 1)
            printf("{\"S\": %d, \"steps\": %lld, \"loop\": %lld, \"per_step\": %.0f, \"lambda\": %.0f, "
                   "\"window\": %.0f, \"entering\": %.0f, \"waitA\": %.0f, \"waitB\": %.0f, "
                   "\"err\": \"%s\"}\n", S, st[0], st[1],
                   double(st[1]) / st[0], double(st[8]) / st[0], double(st[9]) / st[0],
                   double(st[10]) / st[0], double(st[11]) / st[0], double(st[3]) / st[0],
                   cudaGetErrorString(e));
    }
    return 0;
}
