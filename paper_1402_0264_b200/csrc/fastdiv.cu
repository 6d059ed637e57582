// fastdiv.cu -- long division in O(M(n)) by Newton iteration over NTT
// products (the reference's non-goal).
//
// For deg a = na-1 >= deg b = nb-1 and mu = na-nb+1 quotient terms:
//   rb = rev(b) mod X^mu, h = rb^-1 mod X^mu by Newton doubling
//        (h_2k = h_k - X^k * (h_k * e) mod X^k, e = coefficients [k, 2k) of
//         rb * h_k: the low k vanish by construction),
//   rev(q) = rev(a) * h mod X^mu,  r = (a - q*b) mod X^(nb-1).
// Field arithmetic is exact and (q, r) with deg r < deg b is unique, so the
// result is identical to oracle_divmod (oracle.cpp:51-67) -- checked against
// the oracle and the schoolbook kernel in tests/test_gpu_parity.py.
// Products use the NTT (ntt.cu) when both factors are long and the prime has
// the 2-adic roots, else the register-tiled schoolbook kernel (mul.cu).
#include "common.cuh"

namespace mmm_cu {

namespace {

constexpr int FD_T = 256;
constexpr int64_t NTT_MIN = 512;  // shorter factor below this: schoolbook product

// y[i] = x[n-1-i] for i < m (zero where n-1-i < 0)
__global__ void rev_prefix(const uint32_t* __restrict__ x, int64_t n, int64_t m,
                           uint32_t* __restrict__ y) {
    for (int64_t i = int64_t(blockIdx.x) * FD_T + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * FD_T)
        y[i] = (n - 1 - i >= 0) ? x[n - 1 - i] : 0u;
}

// The first Newton doublings, h = rb^-1 mod X^K for K <= BASE_K, in one CTA
// with everything in shared memory (k < BASE_K would otherwise cost ~3 small
// launches per doubling).  Per doubling k -> k2: e[i] = (rb * h)[k + i] =
// sum_{j} rb[j] h[k + i - j] over h's k known terms, then
// h[k + i] = -sum_{j <= i} h[j] e[i - j], i < k2 - k.
constexpr int BASE_K = 512;
__global__ void __launch_bounds__(FD_T) newton_base(const uint32_t* __restrict__ b, int64_t nb,
                                                    int K, uint32_t* __restrict__ h_out,
                                                    FieldParams F) {
    __shared__ uint32_t rb[BASE_K], h[BASE_K], e[BASE_K];
    for (int i = threadIdx.x; i < K; i += FD_T) rb[i] = (nb - 1 - i >= 0) ? b[nb - 1 - i] : 0u;
    __syncthreads();
    if (threadIdx.x == 0) h[0] = invmod(rb[0], F);
    __syncthreads();
    const uint32_t ft = F.fold_terms;
    for (int k = 1; k < K;) {
        const int k2 = min(2 * k, K), n = k2 - k;
        for (int i = threadIdx.x; i < n; i += FD_T) {  // e[i], terms j in [i+1, k+i]
            uint64_t acc = 0;
            uint32_t since = 0;
            for (int j = i + 1; j <= k + i; ++j) {
                if (++since > ft) {
                    acc = fold(acc, F);
                    since = 1;
                }
                acc = mad_wide(rb[j], h[k + i - j], acc);
            }
            e[i] = reduce(acc, F);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += FD_T) {
            uint64_t acc = 0;
            uint32_t since = 0;
            for (int j = 0; j <= i; ++j) {
                if (++since > ft) {
                    acc = fold(acc, F);
                    since = 1;
                }
                acc = mad_wide(h[j], e[i - j], acc);
            }
            h[k + i] = negmod(reduce(acc, F), F);
        }
        __syncthreads();
        k = k2;
    }
    for (int i = threadIdx.x; i < K; i += FD_T) h_out[i] = h[i];
}

// h[k + i] = -t[i], i < n
__global__ void neg_into(const uint32_t* __restrict__ t, int64_t n, uint32_t* __restrict__ h,
                         FieldParams F) {
    for (int64_t i = int64_t(blockIdx.x) * FD_T + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * FD_T)
        h[i] = negmod(t[i], F);
}

// r[i] = a[i] - t[i], i < n
__global__ void sub_into(const uint32_t* __restrict__ a, const uint32_t* __restrict__ t,
                         int64_t n, uint32_t* __restrict__ r, FieldParams F) {
    for (int64_t i = int64_t(blockIdx.x) * FD_T + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * FD_T)
        r[i] = submod(a[i], t[i], F);
}

unsigned blocks_for(int64_t n) {
    return unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, FD_T), 4 * sm_count())));
}

// f[0 .. na+nb-1) = a * b
void product(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb,
             uint32_t* f, cudaStream_t st) {
    if (std::min(na, nb) >= NTT_MIN && ntt_supported(F.p, na + nb - 1))
        launch_ntt_mul(F, a, na, b, nb, f, st);
    else
        launch_mul(F, a, na, b, nb, f, 8, 0, st);
}

}  // namespace

void launch_divmod_fast(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b,
                        int64_t nb, uint32_t* q, uint32_t* r, cudaStream_t st) {
    const int64_t mu = na - nb + 1;
    Scratch sc(st);
    const int64_t nrb = std::min(nb, mu);
    uint32_t* rb = sc.get<uint32_t>(size_t(nrb));
    uint32_t* h = sc.get<uint32_t>(size_t(mu));
    uint32_t* ra = sc.get<uint32_t>(size_t(mu));
    uint32_t* t1 = sc.get<uint32_t>(size_t(2 * std::max(mu, nb)));
    uint32_t* t2 = sc.get<uint32_t>(size_t(2 * mu));
    rev_prefix<<<blocks_for(nrb), FD_T, 0, st>>>(b, nb, nrb, rb);
    check_launch("rev_prefix", dim3(blocks_for(nrb)), dim3(FD_T));
    const int K0 = int(std::min<int64_t>(mu, BASE_K));
    newton_base<<<1, FD_T, 0, st>>>(b, nb, K0, h, F);
    check_launch("newton_base", dim3(1), dim3(FD_T));
    for (int64_t k = K0; k < mu;) {
        const int64_t k2 = std::min(2 * k, mu), nr = std::min(k2, nrb);
        // e = coefficients [k, k2) of rb[0:k2] * h[0:k]
        product(F, rb, nr, h, k, t1, st);
        if (nr + k - 1 <= k) {  // rb shorter than k+1 terms: e = 0, h stays (b constant)
            MMM_CUDA(cudaMemsetAsync(h + k, 0, size_t(k2 - k) * 4, st));
        } else {
            const int64_t ne = std::min(k2, nr + k - 1) - k;  // nonzero part of e
            product(F, h, k, t1 + k, ne, t2, st);
            neg_into<<<blocks_for(k2 - k), FD_T, 0, st>>>(t2, k2 - k, h + k, F);
            check_launch("neg_into", dim3(blocks_for(k2 - k)), dim3(FD_T));
            // t2 holds k + ne - 1 >= k2 - k terms when ne == k2 - k; pad otherwise
            if (k + ne - 1 < k2 - k)
                MMM_CUDA(cudaMemsetAsync(h + k + (k + ne - 1), 0,
                                         size_t(k2 - k - (k + ne - 1)) * 4, st));
        }
        k = k2;
    }
    // rev(q) = rev(a)[0:mu] * h mod X^mu, q = rev(rev(q))
    rev_prefix<<<blocks_for(mu), FD_T, 0, st>>>(a, na, mu, ra);
    check_launch("rev_prefix", dim3(blocks_for(mu)), dim3(FD_T));
    product(F, ra, mu, h, mu, t2, st);
    rev_prefix<<<blocks_for(mu), FD_T, 0, st>>>(t2, mu, mu, q);
    check_launch("rev_prefix", dim3(blocks_for(mu)), dim3(FD_T));
    // r = (a - q * b) mod X^(nb-1)
    if (nb > 1) {
        if (std::min(mu, nb) >= NTT_MIN && ntt_supported(F.p, mu + nb - 1))
            launch_ntt_mul(F, q, mu, b, nb, t1, st);  // long factors: whole NTT product
        else
            launch_mul_range(F, q, mu, b, nb, 0, nb - 1, t1, 8, 0, st);  // low nb-1 only
        sub_into<<<blocks_for(nb - 1), FD_T, 0, st>>>(a, t1, nb - 1, r, F);
        check_launch("sub_into", dim3(blocks_for(nb - 1)), dim3(FD_T));
    }
}

}  // namespace mmm_cu
