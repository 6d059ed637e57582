// pair_bench.cu -- cycles per fused pair of the GCD steady state in isolation
// (registers only: no log, no loop control), to separate the arithmetic's
// latency/issue cost from the chain's bookkeeping.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/pair_bench tools/pair_bench.cu
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

template <int V>
__global__ void kern(const uint32_t* rnd, long long* out, uint32_t* sink, int iters, FieldParams F) {
    const int lane = threadIdx.x & 31;
    const Fld f{F.p, F.pinv};
    uint32_t u[GE], v[GE];
    for (int e = 0; e < GE; ++e) {
        u[e] = rnd[e * 32 + lane] % F.p | 1u;
        v[e] = rnd[64 + e * 32 + lane] % F.p | 1u;
    }
    uint32_t u0 = from_lane(u[0], 0), u1 = from_lane(u[0], 1), u2 = from_lane(u[0], 2),
             u3 = from_lane(u[0], 3);
    uint32_t v0 = from_lane(v[0], 0), v1 = from_lane(v[0], 1), v2 = from_lane(v[0], 2),
             v3 = from_lane(v[0], 3);
    uint32_t acc = 0;
    __syncwarp();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (V == 0) {
            PairOut o;
            if (!fused_pair_la(u, v, u0, u1, u2, u3, v0, v1, v2, v3, f, o)) acc += 1;
            acc += o.ga2;
        } else if (V == 1) {
            uint32_t al, be, ga;
            if (!fused_la(u, v, u0, u1, u2, u3, v0, v1, v2, v3, f, al, be, ga)) acc += 1;
            if (!fused_la(v, u, v0, v1, v2, v3, u0, u1, u2, u3, f, al, be, ga)) acc += 1;
            acc += ga;
        } else if (V == 3) {  // pair with the vector shifts replaced by identity (no SHFL/SEL)
            using A = Arith<0>;
            const uint32_t p = f.p;
            uint32_t nu[GE], nv[GE];
            const uint32_t nx = A::neg(u0, p);
            const uint32_t cc1 = A::comb(v0, u1, nx, v1, f);
            const uint32_t al1 = A::mont(v0, v0, f), be1 = A::mont(v0, nx, f);
            const uint32_t ga1 = A::canon(A::neg(cc1, p), p);
            const uint32_t n0 = A::comb3(al1, u2, be1, v2, ga1, v1, f);
            const uint32_t n1 = A::comb3(al1, u3, be1, v3, ga1, v2, f);
#pragma unroll
            for (int e = 0; e < GE; ++e) nu[e] = A::comb3(al1, u[e], be1, v[e], ga1, v[e] ^ 1u, f);
            const uint32_t n2 = from_lane(nu[0], 2), n3 = from_lane(nu[0], 3);
            const uint32_t ny = A::neg(v0, p);
            const uint32_t cc2 = A::comb(n0, v1, ny, n1, f);
            const uint32_t al2 = A::mont(n0, n0, f), be2 = A::mont(n0, ny, f);
            const uint32_t ga2 = A::canon(A::neg(cc2, p), p);
            const uint32_t m0 = A::comb3(al2, v2, be2, n2, ga2, n1, f);
            const uint32_t m1 = A::comb3(al2, v3, be2, n3, ga2, n2, f);
#pragma unroll
            for (int e = 0; e < GE; ++e) nv[e] = A::comb3(al2, v[e], be2, nu[e], ga2, nu[e] ^ 1u, f);
            const uint32_t m2 = from_lane(nv[0], 2), m3 = from_lane(nv[0], 3);
            if (!(A::nz(cc1, p) & A::nz(n0, p) & A::nz(cc2, p) & A::nz(m0, p))) acc += 1;
            for (int e = 0; e < GE; ++e) { u[e] = nu[e]; v[e] = nv[e]; }
            u0 = n0, u1 = n1, u2 = n2, u3 = n3;
            v0 = m0, v1 = m1, v2 = m2, v3 = m3;
        } else if (V == 4) {  // pair, scalars only + broadcasts from a cheap vector
            using A = Arith<0>;
            const uint32_t p = f.p;
            const uint32_t nx = A::neg(u0, p);
            const uint32_t cc1 = A::comb(v0, u1, nx, v1, f);
            const uint32_t al1 = A::mont(v0, v0, f), be1 = A::mont(v0, nx, f);
            const uint32_t ga1 = A::canon(A::neg(cc1, p), p);
            const uint32_t n0 = A::comb3(al1, u2, be1, v2, ga1, v1, f);
            const uint32_t n1 = A::comb3(al1, u3, be1, v3, ga1, v2, f);
            u[0] += ga1;
            const uint32_t n2 = from_lane(u[0], 2), n3 = from_lane(u[0], 3);
            const uint32_t ny = A::neg(v0, p);
            const uint32_t cc2 = A::comb(n0, v1, ny, n1, f);
            const uint32_t al2 = A::mont(n0, n0, f), be2 = A::mont(n0, ny, f);
            const uint32_t ga2 = A::canon(A::neg(cc2, p), p);
            const uint32_t m0 = A::comb3(al2, v2, be2, n2, ga2, n1, f);
            const uint32_t m1 = A::comb3(al2, v3, be2, n3, ga2, n2, f);
            v[0] += ga2;
            const uint32_t m2 = from_lane(v[0], 2), m3 = from_lane(v[0], 3);
            if (!(A::nz(cc1, p) & A::nz(n0, p) & A::nz(cc2, p) & A::nz(m0, p))) acc += 1;
            u0 = n0, u1 = n1, u2 = n2, u3 = n3;
            v0 = m0, v1 = m1, v2 = m2, v3 = m3;
        } else {  // scalar chain only: cc -> ga -> n0, n1
            using A = Arith<0>;
            const uint32_t nx = A::neg(u0, f.p);
            const uint32_t cc = A::comb(v0, u1, nx, v1, f);
            const uint32_t al = A::mont(v0, v0, f), be = A::mont(v0, nx, f);
            const uint32_t ga = A::canon(A::neg(cc, f.p), f.p);
            const uint32_t n0 = A::comb3(al, u2, be, v2, ga, v1, f);
            const uint32_t n1 = A::comb3(al, u3, be, v3, ga, v2, f);
            u0 = v0; u1 = v1; u2 = v2; u3 = v3;
            v0 = n0; v1 = n1; v2 = n0 ^ 5u; v3 = n1 ^ 3u;
        }
    }
    __syncwarp();
    const long long t = clock64() - t0;
    if (lane == 0) out[V] = t;
    sink[threadIdx.x] = acc ^ u[0] ^ v[GE - 1] ^ u0 ^ v3;
}

int main() {
    const FieldParams F = make_field(469762049u);
    uint32_t *rnd, *sink;
    long long* out;
    cudaMallocManaged(&rnd, 4096 * 4);
    cudaMallocManaged(&out, 128);
    cudaMalloc(&sink, 4096);
    uint64_t x = 88172645463325252ull;
    for (int i = 0; i < 4096; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        rnd[i] = uint32_t(x);
    }
    const int it = 4000;
    for (int rep = 0; rep < 2; ++rep) {
        kern<0><<<1, 32>>>(rnd, out, sink, it, F);
        kern<1><<<1, 32>>>(rnd, out, sink, it, F);
        kern<2><<<1, 32>>>(rnd, out, sink, it, F);
        kern<3><<<1, 32>>>(rnd, out, sink, it, F);
        kern<4><<<1, 32>>>(rnd, out, sink, it, F);
        cudaDeviceSynchronize();
    }
    printf("{\"pair_la_cycles_per_fused\": %.1f, \"two_fused_la_cycles_per_fused\": %.1f, "
           "\"scalar_only_per_fused\": %.1f, \"pair_noshfl\": %.1f, \"pair_scalar_bcast\": %.1f}\n",
           out[0] / (2.0 * it), out[1] / (2.0 * it), out[2] / double(it), out[3] / (2.0 * it), out[4] / (2.0 * it));
    return 0;
}
