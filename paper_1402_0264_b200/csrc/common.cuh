// common.cuh -- host-side plumbing shared by the kernel translation units:
// status propagation, the launch counter behind mmm_cu_launch_count(), and
// stream-ordered scratch memory.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <new>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "field.cuh"

namespace mmm_cu {

// Maps 1:1 onto mmm_status (include/mmm_cu.h).
struct Error : std::runtime_error {
    int status;
    Error(int st, const std::string& m) : std::runtime_error(m), status(st) {}
};
constexpr int ST_INVALID = 1, ST_DOMAIN = 2, ST_CUDA = 3, ST_NCCL = 4, ST_SIM = 5;

// The message behind mmm_last_error() (thread-local, capi.cu).
void set_last_error(const std::string& m);

// Runs one C-ABI entry point: exceptions become an mmm_status plus the
// thread's last-error message.
template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.status;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return ST_INVALID;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return ST_SIM;
    }
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(ST_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define MMM_CUDA(x) ::mmm_cu::cuda_check((x), #x)
#define MMM_LAUNCHED(n) ::mmm_cu::note_launch(n)

// Every kernel launch of this library bumps this counter (bench.py reports
// the number inside its timed region as gpu_launches).
extern std::atomic<uint64_t> g_launches;
inline void note_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
// The calling thread's launch log since the last schedule_reset(): what the
// drop-in reports as SimReport.kernels (name, blocks, threads per block).
void schedule_record(const char* what, dim3 grid, dim3 block);
void schedule_reset();
inline void check_launch(const char* what, dim3 grid = dim3(0, 0, 0), dim3 block = dim3(0, 0, 0)) {
    note_launch();
    cuda_check(cudaGetLastError(), what);
    schedule_record(what, grid, block);
}

// Stream-ordered scratch from a per-(host thread, device) arena: a list of
// device chunks (cudaMallocAsync), handed out by a bump pointer that each
// Scratch restores on destruction (LIFO, nested Scratch objects included).  In
// steady state a call makes no allocation API call (a dozen
// cudaMallocAsync/cudaFreeAsync pairs per GCD call showed up in e2e).
// Reuse across streams is ordered by an event: the outermost Scratch waits on
// the event its predecessor recorded when it was released, so a call on
// another stream (or on a recycled stream handle) never overwrites memory that
// queued work still uses.  The arena belongs to its thread and is freed when
// the thread exits (or by mmm_cu_release_scratch()).
struct Arena {
    std::vector<std::pair<char*, size_t>> chunks;
    size_t ci = 0, off = 0;  // current chunk, offset in it
    int depth = 0;           // live Scratch objects
    cudaEvent_t last = nullptr;  // recorded when the outermost Scratch is released
};
Arena& arena_for();  // the calling thread's arena on the current device
struct Scratch {
    cudaStream_t stream;
    Arena* arena;
    size_t ci0, off0;
    explicit Scratch(cudaStream_t s);
    ~Scratch();
    void* get_bytes(size_t bytes);
    template <class T>
    T* get(size_t count) {
        if (count == 0) count = 1;
        return static_cast<T*>(get_bytes(count * sizeof(T)));
    }
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
};

// A zero-filled device buffer that kernels leave zeroed (the product's split-k
// accumulator and arrival counters), one per (host thread, device).  acquire()
// orders the stream after the buffer's previous user (event); release() marks
// the stream's use.  Growing frees the old buffer in stream order.
struct ZeroBuf {
    unsigned long long* p = nullptr;
    size_t words = 0;
    cudaEvent_t last = nullptr;
};
unsigned long long* zero_buf_acquire(size_t words, cudaStream_t st);
void zero_buf_release(cudaStream_t st);
// Frees every NTT plan (ntt.cu); the caller guarantees no queued work uses one.
void release_plans();

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Fan-out outputs: a kernel stores each output word into every pointer of the
// set (same layout behind each).  With the pointers of other GPUs' buffers
// (symmetric / IPC-mapped memory over NVLink) this is an all-gather fused into
// the producing kernel's epilogue: no gather collective after it.
constexpr int MMM_MAX_FAN = 8;
struct Fan {
    uint32_t* p[MMM_MAX_FAN];
    int n;
};
inline Fan fan_of(uint32_t* f) {
    Fan o{};
    o.p[0] = f;
    o.n = 1;
    return o;
}
inline Fan fan_offset(Fan o, int64_t words) {
    for (int q = 0; q < o.n; ++q) o.p[q] += words;
    return o;
}
#ifdef __CUDACC__
// FAN = false: the single-output instantiation (no extra registers on the hot path)
template <bool FAN>
__device__ __forceinline__ void fan_store(const Fan& o, int64_t i, uint32_t v) {
    if constexpr (!FAN) {
        o.p[0][i] = v;
        return;
    }
    o.p[0][i] = v;
#pragma unroll
    for (int q = 1; q < MMM_MAX_FAN; ++q)  // static indices: the pointers stay kernel parameters
        if (q < o.n) o.p[q][i] = v;
}
#endif

#ifdef __CUDACC__
// Spin until *p >= target, then acquire.  The polling loads are relaxed: an
// ld.acquire.gpu compiles to LDG.STRONG.GPU + CCTL.IVALL, i.e. it invalidates
// the SM's L1 on every spin iteration, and every local-memory or L1-cached
// access of the CTA behind it then goes to L2 (measured: 41 % of the division
// pipeline's stall samples).  One acquiring load after success orders what
// follows (a fence.acq_rel would also wait for the thread's pending stores).
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned spin_until_geq(const unsigned* p, unsigned target) {
    while (ld_relaxed_gpu(p) < target) {
    }
    unsigned v;  // one acquiring load (no MEMBAR, unlike a fence): the value is >= target
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Same, ordering by a full fence after the spin (the division pipeline's bulk
// CTAs measured 5 % faster with it: the fence also drains their own stores).
__device__ __forceinline__ unsigned spin_until_geq_fence(const unsigned* p, unsigned target) {
    unsigned v;
    while ((v = ld_relaxed_gpu(p)) < target) {
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    return v;
}
#endif
inline int sm_count() {
    static int n = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    return n;
}

// ---- launchers (device pointers, async on `st`; outputs untrimmed) --------
// multiplication: f[0 .. na+nb-1) = a * b.  s/l are tile hints (mul.cu).
void launch_mul_range(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b,
                      int64_t nb, int64_t klo, int64_t khi, uint32_t* f, int64_t s, int64_t l,
                      cudaStream_t st);
void launch_mul(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb,
                uint32_t* f, int64_t s, int64_t l, cudaStream_t st);
void launch_mul_batched(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                        const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, uint32_t* Fo,
                        int64_t ldf, int64_t s, cudaStream_t st);
// tensor-core batched product (tcmul.cu): na, nb <= 4096, exact like launch_mul_batched.
// s <= 0 = auto (tensor core where it pays); s >= 1 = the s-parameterised CUDA-core kernel
bool tc_route(const char* env, int64_t s, bool shape_ok, bool worth);
bool tcmul_supported(int64_t na, int64_t nb, int64_t count, int64_t s);
void launch_tcmul_batched(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                          const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, Fan Fo,
                          int64_t ldf, cudaStream_t st);
// one large product on the tensor core, split over the SMs (tcmul.cu)
bool tcmul_single_supported(int64_t na, int64_t nb, int64_t s);
void launch_tcmul_single(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b,
                         int64_t nb, Fan Fo, cudaStream_t st);
// tensor-core batched division (tcdiv.cu): 2 <= nb <= 4096, nb <= na <= 8192.
bool tcdiv_supported(int64_t na, int64_t nb, int64_t count, int64_t s);
void launch_tcdiv_batched(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                          const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, Fan Q,
                          int64_t ldq, Fan R, int64_t ldr, cudaStream_t st);
// division: q[0 .. na-nb+1), r[0 .. nb-1).  b[nb-1] != 0, na >= nb >= 1.
void launch_divmod(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b,
                   int64_t nb, uint32_t* q, uint32_t* r, int64_t s, cudaStream_t st);
void launch_divmod_batched(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                           const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, uint32_t* Q,
                           int64_t ldq, uint32_t* R, int64_t ldr, int64_t s, cudaStream_t st);
// Fan-out variants (outputs stored into every pointer of the set; see Fan).
void launch_mul_range_fan(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b,
                          int64_t nb, int64_t klo, int64_t khi, Fan f, int64_t s, int64_t l,
                          cudaStream_t st);
void launch_mul_batched_fan(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                            const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, Fan Fo,
                            int64_t ldf, int64_t s, cudaStream_t st);
void launch_divmod_batched_fan(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                               const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, Fan Q,
                               int64_t ldq, Fan Rr, int64_t ldr, int64_t s, cudaStream_t st);
// n words of src into every pointer of the fan (capi.cu: fanout_copy_kernel).
void launch_fanout_copy(const uint32_t* src, int64_t n, Fan dst, cudaStream_t st);
// division by Newton iteration over NTT products (fastdiv.cu): same q, r.
void launch_divmod_fast(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b,
                        int64_t nb, uint32_t* q, uint32_t* r, cudaStream_t st);
// gcd: g (capacity max(na,nb)) = monic gcd, *d_ng = its length.
void launch_gcd(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb,
                uint32_t* g, int64_t* d_ng, int64_t s, cudaStream_t st);
// NTT product: f[0 .. na+nb-1).  Requires 2-adic roots of the needed length.
bool ntt_supported(uint32_t p, int64_t out_len);
void launch_ntt_mul(const FieldParams& F, const uint32_t* a, int64_t na, const uint32_t* b,
                    int64_t nb, uint32_t* f, cudaStream_t st);
// sharded four-step NTT product phases (ntt.cu); N = n1 * n2 for nf outputs
void ntt_shape(uint32_t p, int64_t nf, int64_t* n1, int64_t* n2);
void launch_ntt_phase(const FieldParams& F, int phase, const uint32_t* a, int64_t na,
                      const uint32_t* b, int64_t nb, int64_t start, int64_t n, uint32_t* work_a,
                      uint32_t* work_b, uint32_t* f, cudaStream_t st);
void launch_ntt_mul_batched(const FieldParams& F, const uint32_t* A, int64_t lda, int64_t na,
                            const uint32_t* B, int64_t ldb, int64_t nb, int64_t count,
                            uint32_t* Fo, int64_t ldf, cudaStream_t st);

}  // namespace mmm_cu
