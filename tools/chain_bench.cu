// chain_bench.cu -- bisect the cost of one GCD chain fast-path step (one warp,
// synthetic data): comb only, + head shuffle, + window shift, + log store.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/chain_bench tools/chain_bench.cu
#include <cstdint>
#include <cstdio>

constexpr int GE = 4;
constexpr int N = 8192;

__device__ __forceinline__ uint32_t comb(uint32_t y, uint32_t a, uint32_t nx, uint32_t b,
                                         uint32_t p, uint32_t pinv) {
    const uint64_t t = uint64_t(y) * a + uint64_t(nx) * b;
    const uint32_t m = uint32_t(t) * pinv;
    return uint32_t(t >> 32) - __umulhi(m, p) + p;
}

template <int VARIANT>
__global__ void k(const uint32_t* in, long long* out, uint32_t* sink, uint4* logbuf) {
    __shared__ uint4 lg[2048];
    const int lane = threadIdx.x & 31;
    const uint32_t p = 469762049u, pinv = 469762049u * 0 + in[40] | 1u;
    uint32_t u[GE], v[GE];
    for (int e = 0; e < GE; ++e) {
        u[e] = in[(lane + e) & 31] % p + 1;
        v[e] = in[(lane + 7 * e) & 31] % p + 1;
    }
    uint32_t hu = __shfl_sync(~0u, u[0], 0), hv = __shfl_sync(~0u, v[0], 0);
    int du = 100000, dv = 99999, F = 1 << 30;
    long long t0 = clock64();
    for (int s = 0; s < N; ++s) {
        if (VARIANT >= 4 && du < dv) {  // role swap
#pragma unroll
            for (int e = 0; e < GE; ++e) {
                uint32_t t = u[e];
                u[e] = v[e];
                v[e] = t;
            }
            int t = du; du = dv; dv = t;
            uint32_t h = hu; hu = hv; hv = h;
        }
        const uint32_t x = hu, y = hv, nx = 2 * p - x;
#pragma unroll
        for (int e = 0; e < GE; ++e) u[e] = comb(y, u[e], nx, v[e], p, pinv);
        if (VARIANT >= 1) {
            const uint32_t h1 = __shfl_sync(~0u, u[0], 1);
            if (h1 != 0u && h1 != p) {
                if (VARIANT >= 2) {
                    uint32_t r[GE];
#pragma unroll
                    for (int e = 0; e < GE; ++e) r[e] = __shfl_sync(~0u, u[e], (lane + 1) & 31);
#pragma unroll
                    for (int e = 0; e < GE; ++e) u[e] = lane == 31 ? (e + 1 < GE ? r[e + 1] : 0u) : r[e];
                }
                hu = h1;
                --F;
            } else {
                hu = x + 1;
            }
        } else {
            hu = u[0] ^ x;
        }
        du -= 1;
        if (VARIANT >= 3 && lane == 0) {
            const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(lg + (s & 2047)));
            asm volatile("st.volatile.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x),
                         "r"(y), "r"(1u), "r"(unsigned(s + 1))
                         : "memory");
        }
        if (F == 0) break;
    }
    long long t1 = clock64();
    if (lane == 0) out[VARIANT] = t1 - t0;
    uint32_t acc = hu + hv + du + dv;
    for (int e = 0; e < GE; ++e) acc += u[e] + v[e];
    sink[lane] = acc;
    if (lane == 0) logbuf[0] = lg[2047];
}

int main() {
    uint32_t* in;
    long long* out;
    uint32_t* sink;
    uint4* lb;
    cudaMallocManaged(&in, 256);
    cudaMallocManaged(&out, 64);
    cudaMalloc(&sink, 128);
    cudaMalloc(&lb, 64);
    for (int i = 0; i < 64; ++i) in[i] = 0x9e3779b9u * (i + 1);
    auto run = [&](auto kern) {
        kern<<<1, 32>>>(in, out, sink, lb);
        cudaDeviceSynchronize();
        kern<<<1, 32>>>(in, out, sink, lb);
        cudaDeviceSynchronize();
    };
    run(k<0>);
    run(k<1>);
    run(k<2>);
    run(k<3>);
    run(k<4>);
    const char* names[] = {"comb_only", "+head_shfl", "+shift1", "+log_sts128", "+role_swap"};
    printf("{");
    for (int i = 0; i < 5; ++i) printf("%s\"%s\": %.1f", i ? ", " : "", names[i], double(out[i]) / N);
    printf("}\n");
    return 0;
}
