// chain_bench2.cu -- cycles per elimination of the real GCD chain (run_chain
// from paper_1402_0264_b200/csrc/gcd.cu) on synthetic top windows, one warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/chain_bench2 tools/chain_bench2.cu
#include "../paper_1402_0264_b200/csrc/gcd.cu"

namespace mmm_cu {
std::atomic<uint64_t> g_launches{0};
Scratch::Scratch(cudaStream_t s) : stream(s) {}
Scratch::~Scratch() {}
}  // namespace mmm_cu

using namespace mmm_cu;

__global__ void bench(const uint32_t* rnd, long long* out, int batches, FieldParams F) {
    __shared__ uint32_t winA[W1], winB[W1];
    __shared__ __align__(16) StepLog log[LOGCAP];
    __shared__ volatile int done;
    __shared__ BatchMeta c;
    long long steps = 0, cycles = 0;
    for (int bt = 0; bt < batches; ++bt) {
        for (int i = threadIdx.x; i < W1; i += 32) {
            winA[i] = rnd[(bt * 131 + i) & 4095] % F.p;
            winB[i] = rnd[(bt * 137 + i + 2048) & 4095] % F.p;
        }
        if (threadIdx.x == 0) {
            winA[0] |= 1u;  // nonzero leads
            winB[0] |= 1u;
            c.da1 = 100000;
            c.db1 = 99999;
            c.dividend_a = 1;
            done = 0;
        }
        __syncwarp();
        const long long t0 = clock64();
        run_chain<0>(c, log, &done, 1 << 20, Fld{F.p, F.pinv}, winA, winB);
        __syncwarp();
        cycles += clock64() - t0;
        steps += c.steps;
    }
    if (threadIdx.x == 0) {
        out[0] = cycles;
        out[1] = steps;
    }
}

int main() {
    const FieldParams F = make_field(469762049u);
    uint32_t* rnd;
    long long* out;
    cudaMallocManaged(&rnd, 4096 * 4);
    cudaMallocManaged(&out, 16);
    uint64_t x = 88172645463325252ull;
    for (int i = 0; i < 4096; ++i) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        rnd[i] = uint32_t(x);
    }
    bench<<<1, 32>>>(rnd, out, 20, F);
    cudaDeviceSynchronize();
    bench<<<1, 32>>>(rnd, out, 200, F);
    cudaDeviceSynchronize();
    printf("{\"chain_cycles_per_step\": %.1f, \"steps\": %lld, \"GE\": %d}\n",
           double(out[0]) / double(out[1]), out[1], GE);
    return 0;
}
