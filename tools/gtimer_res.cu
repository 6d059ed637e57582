#include <cstdio>
__global__ void k(long long* out) {
    long long prev, t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
    long long c0 = clock64();
    int n = 0;
    while (n < 16) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t != prev) { out[n++] = t - prev; out[16 + n - 1] = clock64() - c0; prev = t; }
    }
}
int main() {
    long long* o; cudaMallocManaged(&o, 256);
    k<<<1,1>>>(o); cudaDeviceSynchronize();
    for (int i = 0; i < 16; ++i) printf("%lld(%lld) ", o[i], o[16+i]); printf("\n");
}
