// chain_bench2.cu -- cycles per elimination of the real GCD chain (run_chain
// from paper_1402_0264_b200/csrc/gcd.cu) on synthetic top windows, and of the
// matrix replay (run_replay, two warps) over the log it wrote, timed apart.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/chain_bench2 tools/chain_bench2.cu
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

// replay without the polling protocol (all entries present): isolates the
// cost of the arithmetic + shuffles from the hand-off
template <int MODE>
__device__ long long replay_plain(int col, const StepLog* log, int n, Fld f, uint32_t* Pg) {
    const int lane = threadIdx.x & 31;
    uint32_t ra[PE], rb[PE];
    for (int e = 0; e < PE; ++e) ra[e] = rb[e] = 0u;
    if (lane == 0) { if (col == 0) ra[0] = 1u; else rb[0] = 1u; }
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        const uint4 en = reinterpret_cast<const uint4*>(log)[i];
        if (en.w & LOG_UA) replay_entry<MODE>(ra, rb, en, f);
        else replay_entry<MODE>(rb, ra, en, f);
    }
    __syncwarp();
    const long long t = clock64() - t0;
    for (int e = 0; e < PE; ++e) Pg[col * 64 + e * 32 + lane] = ra[e] ^ rb[e];
    return t;
}

__global__ void bench(const uint32_t* rnd, long long* out, uint32_t* Pg, uint64_t* rec, int batches,
                      FieldParams F, int mode) {
    __shared__ volatile int ring_ok;
    __shared__ long long tce, tre;
    if (threadIdx.x == 0) ring_ok = 1 << 30;
    __shared__ uint32_t winA[W1], winB[W1], Ps[4 * PL];
    __shared__ int hi[4];
    __shared__ __align__(16) StepLog log[LOGCAP];
    __shared__ volatile int done;
    __shared__ BatchMeta c;
    const int warp = threadIdx.x >> 5;
    long long steps = 0, cycles = 0, rcycles = 0, entries = 0, pcycles = 0, ccon = 0, rcon = 0;
    for (int bt = 0; bt < batches; ++bt) {
        for (int i = threadIdx.x; i < W1; i += blockDim.x) {
            winA[i] = rnd[(bt * 131 + i) & 4095] % F.p;
            winB[i] = rnd[(bt * 137 + i + 2048) & 4095] % F.p;
        }
        for (int i = threadIdx.x; i < LOGCAP; i += blockDim.x)
            reinterpret_cast<uint4*>(log)[i] = make_uint4(0u, 0u, 0u, 0u);
        if (threadIdx.x == 0) {
            winA[0] |= 1u;  // nonzero leads
            winB[0] |= 1u;
            c.da1 = 100000;
            c.db1 = 99999;
            c.dividend_a = 1;
            done = 0;
        }
        __syncthreads();
        long long t0 = clock64();
        if (warp == 0) run_chain<0>(c, log, &done, bt, 1 << 20, Fld{F.p, F.pinv}, winA, winB);
        __syncthreads();
        cycles += clock64() - t0;
        steps += c.steps;
        entries += (done & 0x3FF) - 1;
        if (warp == 1) {
            const long long r0 = clock64();
            run_replay<0>(0, log, &done, bt, Fld{F.p, F.pinv}, rec, 1u, Ps, hi, &ring_ok);
            __syncwarp();
            rcycles += clock64() - r0;
        } else if (warp == 2) {
            run_replay<0>(1, log, &done, bt, Fld{F.p, F.pinv}, rec, 1u, Ps, hi, &ring_ok);
        }
        __syncthreads();
        if (warp == 1) pcycles += replay_plain<0>(0, log, (done & 0x3FF) - 1, Fld{F.p, F.pinv}, Pg + 256);
        __syncthreads();
        // concurrent, as in the kernel: chain || two replay warps (fresh batch tag)
        for (int i = threadIdx.x; i < LOGCAP; i += blockDim.x)
            reinterpret_cast<uint4*>(log)[i] = make_uint4(0u, 0u, 0u, 0u);
        if (threadIdx.x == 0) {
            c.da1 = 100000;
            c.db1 = 99999;
            c.dividend_a = 1;
            done = 0;
        }
        __syncthreads();
        {
            const long long c0 = clock64();
            if (warp == 0) {
                run_chain<0>(c, log, &done, bt + 1000, 1 << 20, Fld{F.p, F.pinv}, winA, winB);
                if (threadIdx.x == 0) tce = clock64() - c0;
            } else if (warp == 1 || !(mode & 1)) {
                run_replay<0>(warp - 1, log, &done, bt + 1000, Fld{F.p, F.pinv}, rec, 1u, Ps, hi,
                              &ring_ok);
                if (threadIdx.x == 32) tre = clock64() - c0;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                ccon += tce;
                rcon += tre;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && bt == batches - 1) {
            out[4] = hi[0]; out[5] = hi[1]; out[6] = hi[2]; out[7] = hi[3];
            out[8] = c.steps; out[9] = done;
        }
    }
    if (threadIdx.x == 0) {
        out[11] = ccon;
        out[12] = rcon;
        out[0] = cycles;
        out[1] = steps;
        out[3] = entries;
    }
    if (threadIdx.x == 32) {
        out[2] = rcycles;
        out[10] = pcycles;
    }
}

int main() {
    const FieldParams F = make_field(469762049u);
    uint32_t* rnd;
    long long* out;
    uint32_t* Pg;
    cudaMalloc(&Pg, 8 * PL * 4);
    cudaMallocManaged(&rnd, 4096 * 4);
    cudaMallocManaged(&out, 256);
    uint64_t* rec;
    cudaMalloc(&rec, 8 * 4 * PL * 8);
    uint64_t x = 88172645463325252ull;
    for (int i = 0; i < 4096; ++i) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        rnd[i] = uint32_t(x);
    }
    const int mode = getenv("CB_MODE") ? atoi(getenv("CB_MODE")) : 0;
    bench<<<1, 96>>>(rnd, out, Pg, rec, 20, F, mode);
    cudaDeviceSynchronize();
    bench<<<1, 96>>>(rnd, out, Pg, rec, 200, F, mode);
    cudaDeviceSynchronize();
    printf("{\"chain_cycles_per_step\": %.1f, \"replay_cycles_per_step\": %.1f, "
           "\"steps_per_entry\": %.2f, \"steps\": %lld, \"GE\": %d}\n",
           double(out[0]) / double(out[1]), double(out[2]) / double(out[1]),
           double(out[1]) / double(out[3]), out[1], GE);
    printf("plain replay cycles/step %.1f\n", double(out[10]) / double(out[1]));
    printf("concurrent: chain end %.0f, replay end %.0f cycles per batch\n", out[11] / 200.0,
           out[12] / 200.0);
#ifdef GCD_TRACE
    long long tw[LOGCAP], tr[LOGCAP], tq[LOGCAP], ta[LOGCAP], tb[LOGCAP];
    cudaMemcpyFromSymbol(ta, g_ta, sizeof(ta));
    cudaMemcpyFromSymbol(tb, g_tb, sizeof(tb));
    cudaMemcpyFromSymbol(tq, g_tp, sizeof(tq));
    cudaMemcpyFromSymbol(tw, g_tw, sizeof(tw));
    cudaMemcpyFromSymbol(tr, g_tr, sizeof(tr));
    for (int i = 0; i < 32; ++i) printf("entry %d: write %lld seen %lld nx %lld top %lld replay %lld lag %lld\n", i, tw[i] - tw[0], tq[i] - tw[0], ta[i] - tw[0], tb[i] - tw[0], tr[i] - tw[0], tr[i] - tw[i]);
#endif
    printf("hi %lld %lld %lld %lld steps %lld done %lld\n", out[4], out[5], out[6], out[7], out[8], out[9]);
    return 0;
}
