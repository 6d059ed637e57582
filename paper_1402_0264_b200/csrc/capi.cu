// capi.cu -- the extern "C" boundary (include/mmm_cu.h).
//
// Validation and error mapping follow the reference entry points
// (proj/src/oracle.cpp:8-78, proj/src/field.cpp:20-42, run_util.hpp:24-29);
// all arithmetic runs in the sm_100a kernels behind the launch_* functions.
// There is no CPU arithmetic fallback: if the CUDA path fails, the call
// returns MMM_CUDA_ERROR.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>
#include <tuple>
#include <map>
#include <new>
#include <random>
#include <string>

#include "../../include/mmm_cu.h"
#include "common.cuh"

namespace mmm_cu {

std::atomic<uint64_t> g_launches{0};

namespace {

// Everything the library keeps per host thread: per device, the thread's
// stream for the host entry points, its scratch arena and its zero buffer; and
// the pinned staging buffer.  Freed when the thread exits (errors ignored: at
// process exit the CUDA runtime may already be gone) or by
// mmm_cu_release_scratch().
constexpr int MAX_DEV = 64;
struct DevState {
    cudaStream_t stream = nullptr;
    cudaStream_t aux[3] = {nullptr, nullptr, nullptr};  // the batch pipeline: H2D, kernels, D2H
    cudaEvent_t ev[16] = {};
    Arena arena;
    ZeroBuf zero;
    bool used = false;
};
struct ThreadState {
    DevState dev[MAX_DEV];
    std::pair<void*, size_t> pinned{nullptr, 0};
    void release() {
        int cur = -1;
        cudaGetDevice(&cur);
        for (int d = 0; d < MAX_DEV; ++d) {
            DevState& s = dev[d];
            if (!s.used) continue;
            cudaSetDevice(d);
            if (s.arena.last) cudaEventSynchronize(s.arena.last);
            if (s.zero.last) cudaEventSynchronize(s.zero.last);
            if (s.stream) cudaStreamSynchronize(s.stream);
            for (auto& c : s.arena.chunks) cudaFree(c.first);
            if (s.zero.p) cudaFree(s.zero.p);
            if (s.arena.last) cudaEventDestroy(s.arena.last);
            if (s.zero.last) cudaEventDestroy(s.zero.last);
            if (s.stream) cudaStreamDestroy(s.stream);
            for (auto& a : s.aux)
                if (a) cudaStreamDestroy(a);
            for (auto& e : s.ev)
                if (e) cudaEventDestroy(e);
            s = DevState{};
        }
        if (pinned.first) cudaFreeHost(pinned.first);
        pinned = {nullptr, 0};
        if (cur >= 0) cudaSetDevice(cur);
    }
    ~ThreadState() { release(); }
};
thread_local ThreadState t_state;

DevState& dev_state() {
    int dev = 0;
    MMM_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= MAX_DEV) throw Error(ST_CUDA, "device ordinal out of range");
    DevState& s = t_state.dev[dev];
    s.used = true;
    return s;
}

}  // namespace

Arena& arena_for() { return dev_state().arena; }

Scratch::Scratch(cudaStream_t s) : stream(s), arena(&arena_for()) {
    if (arena->depth++ == 0 && arena->last) {
        // order this call after the arena's previous user (maybe another stream)
        cudaError_t e = cudaStreamWaitEvent(stream, arena->last, 0);
        if (e != cudaSuccess) {
            --arena->depth;
            cuda_check(e, "cudaStreamWaitEvent(scratch)");
        }
    }
    ci0 = arena->ci;
    off0 = arena->off;
}

void* Scratch::get_bytes(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    Arena& a = *arena;
    for (;;) {
        if (a.ci < a.chunks.size()) {
            auto& c = a.chunks[a.ci];
            if (a.off + bytes <= c.second) {
                void* p = c.first + a.off;
                a.off += bytes;
                return p;
            }
            ++a.ci;  // the rest of this chunk stays unused until the position unwinds
            a.off = 0;
            continue;
        }
        size_t size = std::max<size_t>(bytes, size_t(4) << 20);
        if (!a.chunks.empty()) size = std::max(size, 2 * a.chunks.back().second);
        void* p = nullptr;
        MMM_CUDA(cudaMallocAsync(&p, size, stream));
        a.chunks.push_back({static_cast<char*>(p), size});
    }
}

Scratch::~Scratch() {
    arena->ci = ci0;
    arena->off = off0;
    if (--arena->depth == 0) {
        if (!arena->last) cudaEventCreateWithFlags(&arena->last, cudaEventDisableTiming);
        if (arena->last) cudaEventRecord(arena->last, stream);
    }
}

unsigned long long* zero_buf_acquire(size_t words, cudaStream_t st) {
    ZeroBuf& b = dev_state().zero;
    if (!b.last) MMM_CUDA(cudaEventCreateWithFlags(&b.last, cudaEventDisableTiming));
    MMM_CUDA(cudaStreamWaitEvent(st, b.last, 0));  // after the buffer's previous user
    if (b.words < words) {
        if (b.p) MMM_CUDA(cudaFreeAsync(b.p, st));  // ordered after that user too
        b.p = nullptr;
        b.words = 0;
        const size_t n = std::max(words, size_t(1) << 16);
        MMM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&b.p), n * sizeof(unsigned long long), st));
        MMM_CUDA(cudaMemsetAsync(b.p, 0, n * sizeof(unsigned long long), st));
        b.words = n;
    }
    return b.p;
}

void zero_buf_release(cudaStream_t st) {
    ZeroBuf& b = dev_state().zero;
    MMM_CUDA(cudaEventRecord(b.last, st));
}

}  // namespace mmm_cu

namespace {
thread_local std::string t_err;
}

namespace mmm_cu {
void set_last_error(const std::string& m) { t_err = m; }

namespace {
struct Schedule {
    std::vector<mmm_kernel_rec> recs;
    int64_t total = 0;
};
thread_local Schedule t_sched;
}  // namespace

void schedule_reset() {
    t_sched.recs.clear();
    t_sched.total = 0;
}

void schedule_record(const char* what, dim3 grid, dim3 block) {
    ++t_sched.total;
    if (t_sched.recs.size() >= 65536) return;  // counted, not kept
    mmm_kernel_rec r{};
    std::strncpy(r.name, what, sizeof(r.name) - 1);
    r.blocks = int64_t(grid.x) * grid.y * grid.z;
    r.threads = int32_t(block.x * block.y * block.z);
    t_sched.recs.push_back(r);
}

__global__ void check_rows_kernel(const uint32_t* __restrict__ d, int64_t rows, int64_t n,
                                  uint32_t p, unsigned* flag) {
    unsigned bad = 0;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const uint32_t* row = d + r * n;
        for (int64_t c = threadIdx.x; c < n; c += blockDim.x) bad |= __ldg(row + c) >= p;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

// validate_coeffs (run_util.hpp:24-29) for one operand where it landed
__global__ void check_flat_kernel(const uint32_t* __restrict__ d, int64_t n, uint32_t p,
                                  unsigned* flag) {
    unsigned bad = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        bad |= __ldg(d + i) >= p;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

}  // namespace mmm_cu

using namespace mmm_cu;

namespace {

// Field::Field (field.cpp:10-25).  The trial-division primality test costs
// ~70 us on the host for a 29-bit p; the calling thread remembers the last
// few primes it validated, so repeated calls (the bench's steps, a batch of
// small products) pay it once.
FieldParams field_or_throw(int64_t p) {
    struct Seen {
        int64_t p = 0;
        FieldParams F{};
    };
    thread_local Seen seen[8];
    thread_local int next_slot = 0;
    for (const Seen& e : seen)
        if (e.p == p && p != 0) return e.F;
    if (p < 2 || p >= (int64_t(1) << 31))
        throw Error(ST_INVALID, "field: p must satisfy 2 <= p < 2^31, got " + std::to_string(p));
    bool prime = p == 2 || (p % 2 != 0);
    for (int64_t d = 3; prime && d * d <= p; d += 2)
        if (p % d == 0) prime = false;
    if (!prime) throw Error(ST_INVALID, "field: p must be prime, got " + std::to_string(p));
    const FieldParams F = make_field(uint32_t(p));
    seen[next_slot] = {p, F};
    next_slot = (next_slot + 1) % 8;
    return F;
}

void check_operand(const uint32_t* c, int64_t n, const char* who) {
    if (n < 0) throw Error(ST_INVALID, std::string(who) + ": negative length");
    if (n > 0 && c == nullptr) throw Error(ST_INVALID, std::string(who) + ": null pointer");
}

// validate_coeffs (run_util.hpp:24-29).
void check_canonical(const uint32_t* c, int64_t n, uint32_t p, const char* who) {
    check_operand(c, n, who);
    // blockwise maximum without an early exit, so the scan vectorises (the
    // branchy per-word test was most of the host time of a large e2e call)
    for (int64_t i0 = 0; i0 < n; i0 += 8192) {
        const int64_t e = std::min<int64_t>(n, i0 + 8192);
        uint32_t m = 0;
        for (int64_t i = i0; i < e; ++i) m = c[i] > m ? c[i] : m;
        if (m >= p)
            throw Error(ST_INVALID,
                        std::string(who) + ": coefficients must be canonical field elements");
    }
}

int64_t trimmed_len(const uint32_t* c, int64_t n) {
    while (n > 0 && c[n - 1] == 0) --n;
    return n;
}

// The calling thread's stream on the current device (created on first use).
cudaStream_t thread_stream() {
    DevState& s = dev_state();
    if (!s.stream) MMM_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    return s.stream;
}

void need_cap(int64_t cap, int64_t need, const char* what) {
    if (cap < need)
        throw Error(ST_INVALID, std::string(what) + ": output capacity " + std::to_string(cap) +
                                    " < " + std::to_string(need));
}

uint32_t* to_device(Scratch& s, const uint32_t* h, int64_t n) {
    uint32_t* d = s.get<uint32_t>(size_t(n));
    if (n) MMM_CUDA(cudaMemcpyAsync(d, h, size_t(n) * 4, cudaMemcpyHostToDevice, s.stream));
    return d;
}

void to_host(uint32_t* h, const uint32_t* d, int64_t n, cudaStream_t st) {
    if (n) MMM_CUDA(cudaMemcpyAsync(h, d, size_t(n) * 4, cudaMemcpyDeviceToHost, st));
}

void sync(cudaStream_t st) { MMM_CUDA(cudaStreamSynchronize(st)); }

// Per-thread pinned host staging (grown on demand, kept): device-to-host reads
// that must complete before the call returns go here, so one synchronisation
// covers them all.
uint32_t* pinned_stage(size_t bytes) {
    auto& buf = t_state.pinned;
    if (buf.second < bytes) {
        if (buf.first) cudaFreeHost(buf.first);
        const size_t n = std::max(bytes, size_t(1) << 20);
        void* p = nullptr;
        MMM_CUDA(cudaMallocHost(&p, n));
        buf = {p, n};
    }
    return static_cast<uint32_t*>(buf.first);
}

// Single host calls with large operands (> 2^18 words together)
// validate them on the device, where they land (a host scan of a 2^20-term
// operand cost more than its copy): one flag per operand, read back with the
// results and reported after the synchronisation (outputs are then
// unspecified, as for any failed call).  Any other error the call raises
// first re-runs the host scan, so a non-canonical operand is still reported
// ahead of it, as validate_coeffs comes first in the reference.  Smaller
// operands are scanned on the host up front (errors before any device work).
constexpr int64_t DEV_CHECK_WORDS = int64_t(1) << 18;
struct DevCheck {
    unsigned* flags = nullptr;
    const char* who[2] = {nullptr, nullptr};
    int n = 0;
    cudaStream_t st;
    DevCheck(Scratch& sc, cudaStream_t s) : st(s) {
        flags = sc.get<unsigned>(2);
        MMM_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned), st));
    }
    void add(const uint32_t* d, int64_t len, uint32_t p, const char* w) {
        if (len > 0) {
            const unsigned blocks = unsigned(std::min<int64_t>(ceil_div(len, 2048), 2LL * sm_count()));
            check_flat_kernel<<<blocks, 256, 0, st>>>(d, len, p, flags + n);
            note_launch();  // counted, but not part of the program's schedule (SimReport)
            cuda_check(cudaGetLastError(), "check_flat_kernel");
        }
        who[n++] = w;
    }
    uint32_t* stage() {  // the flags' copy, with the results
        uint32_t* h = pinned_stage(16);
        MMM_CUDA(cudaMemcpyAsync(h, flags, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        return h;
    }
    void report(const uint32_t* h) const {  // after the synchronisation
        for (int i = 0; i < n; ++i)
            if (h[i])
                throw Error(ST_INVALID,
                            std::string(who[i]) + ": coefficients must be canonical field elements");
    }
};

// A single host call's device part: both operands uploaded and checked where
// they land, `body` launches the kernels and queues the result copies, one
// synchronisation, then the check's verdict.
template <class Body>
void checked_call(cudaStream_t st, bool dev_check, uint32_t p, const uint32_t* a, int64_t na,
                  const char* wa, const uint32_t* b, int64_t nb, const char* wb, Body body) {
    Scratch sc(st);
    const uint32_t* da = to_device(sc, a, na);
    const uint32_t* db = to_device(sc, b, nb);
    DevCheck chk(sc, st);
    if (dev_check) {  // (else the caller scanned on the host)
        chk.add(da, na, p, wa);
        chk.add(db, nb, p, wb);
    }
    body(sc, da, db);
    const uint32_t* h = chk.stage();
    sync(st);
    chk.report(h);
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// ---- pipelined batches (host buffers) --------------------------------------
// A batched host call streams its instances through the GPU in chunks over
// three streams -- copies in, kernels, copies out -- and a ring of device
// slots: chunk k's H2D waits only for the D2H that last used its slot, its
// kernels for its H2D, its D2H for its kernels, so the copy engines run both
// directions while the SMs work on the chunk in between.  The canonical-
// coefficient check (run_util.hpp:24-29) runs on the device as each chunk
// lands -- the host scan of a cfg5 batch (335 MB) cost more than its transfer
// -- and is reported after the join (outputs are then unspecified, as for any
// failed call).  D2H of chunk k is issued after chunk k+1's H2D and kernels,
// so pageable (blocking) copies still overlap.
struct HostIn {
    const uint32_t* p;
    int64_t ld, n;
    const char* what;  // error message subject
};
struct HostOut {
    uint32_t* p;
    int64_t ld, n;
};

constexpr int PIPE_SLOTS = 3;

template <class Launch>
void pipelined_batch(const FieldParams& F, int64_t count, std::vector<HostIn> ins,
                     std::vector<HostOut> outs, Launch launch) {
    DevState& ds = dev_state();
    const cudaStream_t st0 = thread_stream();
    for (auto& a : ds.aux)
        if (!a) MMM_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    for (auto& e : ds.ev)
        if (!e) MMM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const cudaStream_t sH = ds.aux[0], sK = ds.aux[1], sD = ds.aux[2];
    cudaEvent_t* evIn = ds.ev + 1;                // [slot]: chunk's inputs landed
    cudaEvent_t* evOut = evIn + PIPE_SLOTS;       // [slot]: chunk's kernels done
    cudaEvent_t* evFree = evOut + PIPE_SLOTS;     // [slot]: chunk's results copied out
    int64_t row_words = 0;
    for (auto& i : ins) row_words += i.n;
    for (auto& o : outs) row_words += o.n;
    // about 16 chunks per call, each a whole number of CTA rounds (one CTA per SM)
    // and >= 2 MB
    const int64_t sms = sm_count();
    int64_t chunk = ceil_div(ceil_div(count, 16), sms) * sms;
    chunk = std::max<int64_t>(chunk, ceil_div(int64_t(2) << 20, 4 * std::max<int64_t>(row_words, 1)));
    chunk = std::min<int64_t>(chunk, count);
    // the first and last chunks are one CTA round when the batch allows: the first H2D
    // and the last kernels + D2H are the pipeline's unoverlapped fill and drain
    std::vector<int64_t> cuts{0};
    {
        const int64_t edge = std::min(chunk, sms);
        const bool ramp = count >= 2 * edge + 2 * chunk;
        if (ramp) cuts.push_back(edge);
        const int64_t body_end = ramp ? count - edge : count;
        while (cuts.back() < body_end) cuts.push_back(std::min(body_end, cuts.back() + chunk));
        if (ramp) cuts.push_back(count);
    }
    const int64_t nchunks = int64_t(cuts.size()) - 1;
    const int slots = int(std::min<int64_t>(PIPE_SLOTS, nchunks));
    uint32_t* stage = pinned_stage(ins.size() * 4 + 16);
    {
        Scratch sc(st0);
        std::vector<uint32_t*> din[PIPE_SLOTS], dout[PIPE_SLOTS];
        for (int l = 0; l < slots; ++l) {
            for (auto& i : ins) din[l].push_back(sc.get<uint32_t>(size_t(chunk * i.n)));
            for (auto& o : outs) dout[l].push_back(sc.get<uint32_t>(size_t(chunk * std::max<int64_t>(o.n, 1))));
        }
        unsigned* flags = sc.get<unsigned>(ins.size());
        MMM_CUDA(cudaMemsetAsync(flags, 0, ins.size() * sizeof(unsigned), st0));
        MMM_CUDA(cudaEventRecord(ds.ev[0], st0));  // fork: scratch and flags ready
        for (cudaStream_t a : {sH, sK, sD}) MMM_CUDA(cudaStreamWaitEvent(a, ds.ev[0], 0));
        auto d2h = [&](int64_t k) {
            const int l = int(k % slots);
            const int64_t c0 = cuts[k], c = cuts[k + 1] - c0;
            MMM_CUDA(cudaStreamWaitEvent(sD, evOut[l], 0));
            for (size_t j = 0; j < outs.size(); ++j)
                if (outs[j].n)
                    MMM_CUDA(cudaMemcpy2DAsync(outs[j].p + c0 * outs[j].ld, size_t(outs[j].ld) * 4,
                                               dout[l][j], size_t(outs[j].n) * 4,
                                               size_t(outs[j].n) * 4, size_t(c),
                                               cudaMemcpyDeviceToHost, sD));
            MMM_CUDA(cudaEventRecord(evFree[l], sD));
        };
        for (int64_t k = 0; k < nchunks; ++k) {
            const int l = int(k % slots);
            const int64_t c0 = cuts[k], c = cuts[k + 1] - c0;
            if (k >= slots) MMM_CUDA(cudaStreamWaitEvent(sH, evFree[l], 0));  // slot drained
            for (size_t j = 0; j < ins.size(); ++j)
                MMM_CUDA(cudaMemcpy2DAsync(din[l][j], size_t(ins[j].n) * 4, ins[j].p + c0 * ins[j].ld,
                                           size_t(ins[j].ld) * 4, size_t(ins[j].n) * 4, size_t(c),
                                           cudaMemcpyHostToDevice, sH));
            MMM_CUDA(cudaEventRecord(evIn[l], sH));
            MMM_CUDA(cudaStreamWaitEvent(sK, evIn[l], 0));
            for (size_t j = 0; j < ins.size(); ++j) {
                const unsigned blocks = unsigned(std::min<int64_t>(c, 4LL * sm_count()));
                check_rows_kernel<<<blocks, 256, 0, sK>>>(din[l][j], c, ins[j].n, F.p, flags + j);
                check_launch("check_rows_kernel", dim3(blocks), dim3(256));
            }
            launch(din[l], dout[l], c, sK);
            MMM_CUDA(cudaEventRecord(evOut[l], sK));
            if (k > 0) d2h(k - 1);
        }
        d2h(nchunks - 1);
        for (int a = 0; a < 3; ++a) {  // join before the scratch is released
            MMM_CUDA(cudaEventRecord(ds.ev[13 + a], ds.aux[a]));
            MMM_CUDA(cudaStreamWaitEvent(st0, ds.ev[13 + a], 0));
        }
        MMM_CUDA(cudaMemcpyAsync(stage, flags, ins.size() * sizeof(unsigned),
                                 cudaMemcpyDeviceToHost, st0));
    }
    sync(st0);
    for (size_t j = 0; j < ins.size(); ++j)
        if (stage[j])
            throw Error(ST_INVALID, std::string(ins[j].what) +
                                        ": coefficients must be canonical field elements");
}

}  // namespace

struct mmm_rng {
    std::mt19937_64 eng;
};

extern "C" {

const char* mmm_last_error(void) { return t_err.c_str(); }

int mmm_cu_last_schedule(mmm_kernel_rec* out, int32_t cap, int32_t* n) {
    const auto& r = t_sched.recs;
    const int32_t k = int32_t(std::min<size_t>(r.size(), size_t(std::max(cap, 0))));
    if (k && out) std::memcpy(out, r.data(), size_t(k) * sizeof(mmm_kernel_rec));
    if (n) *n = int32_t(std::min<int64_t>(t_sched.total, INT32_MAX));
    return MMM_OK;
}

int mmm_cu_release_scratch(void) {
    return guarded([&] { t_state.release(); });
}

// ---- pinned result pool ------------------------------------------------
namespace {
struct HostPool {
    std::mutex mu;
    std::multimap<size_t, void*> free_;     // rounded size -> buffer
    std::map<void*, size_t> live;           // buffer -> rounded size
    size_t cached = 0;
    static constexpr size_t CAP = size_t(2) << 30;
    static size_t round(size_t b) {  // 1 MB granularity (few distinct sizes per workload)
        const size_t g = size_t(1) << 20;
        return std::max(g, (b + g - 1) / g * g);
    }
    void drain() {
        std::lock_guard<std::mutex> lk(mu);
        for (auto& kv : free_) cudaFreeHost(kv.second);
        free_.clear();
        cached = 0;
    }
} g_hostpool;
}  // namespace

int mmm_cu_host_alloc(size_t bytes, void** out) {
    return guarded([&] {
        if (!out) throw Error(ST_INVALID, "mmm_cu_host_alloc: null out");
        const size_t n = HostPool::round(bytes);
        {
            std::lock_guard<std::mutex> lk(g_hostpool.mu);
            auto it = g_hostpool.free_.find(n);
            if (it != g_hostpool.free_.end()) {
                *out = it->second;
                g_hostpool.cached -= n;
                g_hostpool.free_.erase(it);
                g_hostpool.live[*out] = n;
                return;
            }
        }
        void* p = nullptr;
        MMM_CUDA(cudaMallocHost(&p, n));
        std::lock_guard<std::mutex> lk(g_hostpool.mu);
        g_hostpool.live[p] = n;
        *out = p;
    });
}

int mmm_cu_host_free(void* p) {
    return guarded([&] {
        if (!p) return;
        std::lock_guard<std::mutex> lk(g_hostpool.mu);
        auto it = g_hostpool.live.find(p);
        if (it == g_hostpool.live.end())
            throw Error(ST_INVALID, "mmm_cu_host_free: not a buffer from mmm_cu_host_alloc");
        const size_t n = it->second;
        g_hostpool.live.erase(it);
        if (g_hostpool.cached + n <= HostPool::CAP) {
            g_hostpool.free_.emplace(n, p);
            g_hostpool.cached += n;
        } else {
            MMM_CUDA(cudaFreeHost(p));
        }
    });
}

int mmm_cu_release_all(void) {
    return guarded([&] {
        g_hostpool.drain();
        int n = 0, cur = 0;
        MMM_CUDA(cudaGetDevice(&cur));
        MMM_CUDA(cudaGetDeviceCount(&n));
        for (int d = 0; d < n; ++d) {
            MMM_CUDA(cudaSetDevice(d));
            MMM_CUDA(cudaDeviceSynchronize());
        }
        MMM_CUDA(cudaSetDevice(cur));
        release_plans();
        t_state.release();
    });
}
int mmm_version(void) { return 1; }
uint64_t mmm_cu_launch_count(void) { return g_launches.load(); }

int mmm_field_check(int64_t p) {
    return guarded([&] { field_or_throw(p); });
}

int mmm_field_inv(int64_t a, int64_t p, int64_t* out) {
    return guarded([&] {
        field_or_throw(p);
        if (a < 0 || a >= p) throw Error(ST_INVALID, "field: non-canonical element");
        if (a == 0) throw Error(ST_DOMAIN, "field: inverse of zero");
        // extended Euclid, as Field::inv
        int64_t old_r = a, r = p, old_t = 1, t = 0;
        while (r != 0) {
            int64_t q = old_r / r, tmp = old_r - q * r;
            old_r = r;
            r = tmp;
            tmp = old_t - q * t;
            old_t = t;
            t = tmp;
        }
        old_t %= p;
        *out = old_t < 0 ? old_t + p : old_t;
    });
}

mmm_rng* mmm_rng_create(uint64_t seed) {
    try {
        return new mmm_rng{std::mt19937_64(seed)};
    } catch (...) {
        return nullptr;
    }
}
void mmm_rng_destroy(mmm_rng* g) { delete g; }
uint64_t mmm_rng_next(mmm_rng* g) { return g->eng(); }

int mmm_random_poly(mmm_rng* g, int64_t terms, int64_t p, uint32_t* out) {
    return guarded([&] {
        field_or_throw(p);
        if (terms < 1) throw Error(ST_INVALID, "random_poly: terms must be >= 1");
        std::uniform_int_distribution<std::int64_t> any(0, p - 1);
        std::uniform_int_distribution<std::int64_t> nonzero(1, p - 1);
        for (int64_t i = 0; i + 1 < terms; ++i) out[i] = uint32_t(any(g->eng));
        out[terms - 1] = uint32_t(nonzero(g->eng));
    });
}

// ------------------------------------------------------------ multiply ----
int mmm_cu_mul(int64_t p, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb, int64_t s,
               int64_t l, uint32_t* f, int64_t f_cap, int64_t* nf) {
    return guarded([&] {
        schedule_reset();
        const FieldParams F = field_or_throw(p);
        const char* wa = "multiplication first operand";
        const char* wb = "multiplication second operand";
        check_operand(a, na, wa);
        check_operand(b, nb, wb);
        const int64_t na0 = na, nb0 = nb;
        auto host_scan = [&] {
            check_canonical(a, na0, F.p, wa);
            check_canonical(b, nb0, F.p, wb);
        };
        const bool scanned = na0 + nb0 <= DEV_CHECK_WORDS;
        if (scanned) host_scan();
        *nf = 0;
        na = trimmed_len(a, na);
        nb = trimmed_len(b, nb);
        if (na == 0 || nb == 0) {  // oracle.cpp:9
            host_scan();
            return;
        }
        try {
            need_cap(f_cap, na + nb - 1, "multiplication");
        } catch (Error&) {
            host_scan();
            throw;
        }
        cudaStream_t st = thread_stream();
        checked_call(st, !scanned, F.p, a, na, wa, b, nb, wb,
                     [&](Scratch& sc, const uint32_t* da, const uint32_t* db) {
                         uint32_t* df = sc.get<uint32_t>(size_t(na + nb - 1));
                         launch_mul(F, da, na, db, nb, df, s, l, st);
                         to_host(f, df, na + nb - 1, st);
                     });
        *nf = trimmed_len(f, na + nb - 1);
    });
}

int mmm_cu_mul_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b, int64_t nb,
                   int64_t s, uint32_t* d_f, void* stream) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        if (na < 1 || nb < 1) throw Error(ST_INVALID, "multiplication: operands must be nonzero");
        launch_mul(F, d_a, na, d_b, nb, d_f, s, 0, as_stream(stream));
    });
}

int mmm_cu_mul_range_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b,
                         int64_t nb, int64_t k0, int64_t k1, int64_t s, uint32_t* d_f,
                         void* stream) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        if (na < 1 || nb < 1) throw Error(ST_INVALID, "multiplication: operands must be nonzero");
        if (k0 < 0 || k1 < k0 || k1 > na + nb - 1)
            throw Error(ST_INVALID, "multiplication: output range outside [0, na + nb - 1)");
        launch_mul_range(F, d_a, na, d_b, nb, k0, k1, d_f, s, 0, as_stream(stream));
    });
}

int mmm_cu_mul_batched(int64_t p, const uint32_t* A, int64_t lda, int64_t na, const uint32_t* B,
                       int64_t ldb, int64_t nb, int64_t count, int64_t s, uint32_t* Fo,
                       int64_t ldf) {
    return guarded([&] {
        schedule_reset();
        const FieldParams F = field_or_throw(p);
        if (na < 1 || nb < 1 || count < 0 || lda < na || ldb < nb || ldf < na + nb - 1)
            throw Error(ST_INVALID, "multiplication batch: bad shape");
        if (count == 0) return;
        const int64_t nf = na + nb - 1;
        pipelined_batch(F, count,
                        {{A, lda, na, "multiplication batch first operand"},
                         {B, ldb, nb, "multiplication batch second operand"}},
                        {{Fo, ldf, nf}},
                        [&](const std::vector<uint32_t*>& in, const std::vector<uint32_t*>& out,
                            int64_t c, cudaStream_t st) {
                            launch_mul_batched(F, in[0], na, na, in[1], nb, nb, c, out[0], nf, s, st);
                        });
    });
}

int mmm_cu_mul_batched_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                           const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count, int64_t s,
                           uint32_t* d_F, int64_t ldf, void* stream) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        if (na < 1 || nb < 1 || count < 0 || lda < na || ldb < nb || ldf < na + nb - 1)
            throw Error(ST_INVALID, "multiplication batch: bad shape");
        if (count) launch_mul_batched(F, d_A, lda, na, d_B, ldb, nb, count, d_F, ldf, s,
                                      as_stream(stream));
    });
}

// ------------------------------------------------------------ fan-out -----
// Outputs stored into every buffer of a set (1..MMM_MAX_FAN device pointers,
// same layout): with the buffers of every rank (symmetric / IPC-mapped memory
// over NVLink) the all-gather of a sharded batch is fused into the kernel.
namespace {
Fan fan_or_throw(uint32_t* const* ptrs, int32_t n, const char* what) {
    if (n < 1 || n > MMM_MAX_FAN || ptrs == nullptr)
        throw Error(ST_INVALID, std::string(what) + ": fan-out count must be in [1, " +
                                    std::to_string(MMM_MAX_FAN) + "]");
    Fan f{};
    for (int q = 0; q < n; ++q) {
        if (ptrs[q] == nullptr) throw Error(ST_INVALID, std::string(what) + ": null output");
        f.p[q] = ptrs[q];
    }
    f.n = n;
    return f;
}
}  // namespace

// Push one buffer into every buffer of a fan (the gather for kernels without a
// fan-out epilogue, e.g. the NTT batch): 16-byte loads and stores when every
// pointer is aligned, one pass over the source.
__global__ void fanout_copy_kernel(const uint32_t* __restrict__ src, int64_t n, Fan dst,
                                   bool vec) {
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (vec) {
        const int64_t n4 = n / 4;
        for (; i < n4; i += stride) {
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(src) + i);
#pragma unroll
            for (int q = 0; q < MMM_MAX_FAN; ++q)
                if (q < dst.n) reinterpret_cast<uint4*>(dst.p[q])[i] = v;
        }
        i = 4 * n4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    }
    for (; i < n; i += stride) {
        const uint32_t v = src[i];
#pragma unroll
        for (int q = 0; q < MMM_MAX_FAN; ++q)
            if (q < dst.n) dst.p[q][i] = v;
    }
}

}  // extern "C"

namespace mmm_cu {
void launch_fanout_copy(const uint32_t* src, int64_t n, Fan f, cudaStream_t st) {
    if (n <= 0) return;
    bool vec = reinterpret_cast<uintptr_t>(src) % 16 == 0;
    for (int q = 0; q < f.n; ++q) vec = vec && reinterpret_cast<uintptr_t>(f.p[q]) % 16 == 0;
    const int64_t work = vec ? (n + 3) / 4 : n;
    const unsigned blocks = unsigned(std::min<int64_t>((work + 255) / 256, 8LL * sm_count()));
    fanout_copy_kernel<<<blocks, 256, 0, st>>>(src, n, f, vec);
    check_launch("fanout_copy_kernel", dim3(blocks), dim3(256));
}
}  // namespace mmm_cu

extern "C" {

int mmm_cu_fanout_copy_dev(const uint32_t* d_src, int64_t n, uint32_t* const* d_dst,
                           int32_t n_out, void* stream) {
    return guarded([&] {
        const Fan f = fan_or_throw(d_dst, n_out, "fan-out copy");
        if (n < 0) throw Error(ST_INVALID, "fan-out copy: negative length");
        launch_fanout_copy(d_src, n, f, as_stream(stream));
    });
}

int mmm_cu_mul_range_fanout_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b,
                                int64_t nb, int64_t k0, int64_t k1, int64_t s,
                                uint32_t* const* d_f, int32_t n_out, void* stream) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        const Fan f = fan_or_throw(d_f, n_out, "multiplication");
        if (na < 1 || nb < 1) throw Error(ST_INVALID, "multiplication: operands must be nonzero");
        if (k0 < 0 || k1 < k0 || k1 > na + nb - 1)
            throw Error(ST_INVALID, "multiplication: output range outside [0, na + nb - 1)");
        launch_mul_range_fan(F, d_a, na, d_b, nb, k0, k1, f, s, 0, as_stream(stream));
    });
}

int mmm_cu_mul_batched_fanout_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                                  const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                                  int64_t s, uint32_t* const* d_F, int32_t n_out, int64_t ldf,
                                  void* stream) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        const Fan f = fan_or_throw(d_F, n_out, "multiplication batch");
        if (na < 1 || nb < 1 || count < 0 || lda < na || ldb < nb || ldf < na + nb - 1)
            throw Error(ST_INVALID, "multiplication batch: bad shape");
        if (count)
            launch_mul_batched_fan(F, d_A, lda, na, d_B, ldb, nb, count, f, ldf, s,
                                   as_stream(stream));
    });
}

int mmm_cu_divmod_batched_fanout_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                                     const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                                     int64_t s, uint32_t* const* d_Q, int64_t ldq,
                                     uint32_t* const* d_R, int64_t ldr, int32_t n_out,
                                     void* stream) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        const Fan q = fan_or_throw(d_Q, n_out, "division batch");
        const Fan r = fan_or_throw(d_R, n_out, "division batch");
        if (nb < 1 || na < nb || count < 0 || lda < na || ldb < nb || ldq < na - nb + 1 ||
            ldr < nb - 1)
            throw Error(ST_INVALID, "division batch: bad shape");
        if (count)
            launch_divmod_batched_fan(F, d_A, lda, na, d_B, ldb, nb, count, q, ldq, r, ldr, s,
                                      as_stream(stream));
    });
}

// ------------------------------------------------------------- divmod -----
int mmm_cu_divmod(int64_t p, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb,
                  int64_t s, uint32_t* q, int64_t q_cap, int64_t* nq, uint32_t* r, int64_t r_cap,
                  int64_t* nr) {
    return guarded([&] {
        schedule_reset();
        const FieldParams F = field_or_throw(p);
        const char* wa = "division dividend";
        const char* wb = "division divisor";
        check_operand(a, na, wa);
        check_operand(b, nb, wb);
        const int64_t na0 = na;
        auto host_scan = [&] {  // the paths below that raise or return before the device
            check_canonical(a, na0, F.p, wa);
            check_canonical(b, nb, F.p, wb);
        };
        const bool scanned = na0 + nb <= DEV_CHECK_WORDS;
        if (scanned) host_scan();
        *nq = *nr = 0;
        // oracle.cpp:52-55: b is used as given; a is trimmed.
        try {
            if (nb == 0) throw Error(ST_DOMAIN, "divmod: division by the zero polynomial");
            na = trimmed_len(a, na);
            if (na < nb) {
                host_scan();
                need_cap(r_cap, na, "division remainder");
                if (na) std::memcpy(r, a, size_t(na) * 4);
                *nr = na;
                return;
            }
            if (b[nb - 1] == 0) throw Error(ST_DOMAIN, "field: inverse of zero");
            need_cap(q_cap, na - nb + 1, "division quotient");
            need_cap(r_cap, nb - 1, "division remainder");
        } catch (Error&) {
            host_scan();
            throw;
        }
        cudaStream_t st = thread_stream();
        checked_call(st, !scanned, F.p, a, na, wa, b, nb, wb,
                     [&](Scratch& sc, const uint32_t* da, const uint32_t* db) {
                         uint32_t* dq = sc.get<uint32_t>(size_t(na - nb + 1));
                         uint32_t* dr = sc.get<uint32_t>(size_t(nb));
                         launch_divmod(F, da, na, db, nb, dq, dr, s, st);
                         to_host(q, dq, na - nb + 1, st);
                         to_host(r, dr, nb - 1, st);
                     });
        *nq = trimmed_len(q, na - nb + 1);
        *nr = trimmed_len(r, nb - 1);
    });
}

int mmm_cu_ntt_shape(int64_t p, int64_t nf, int64_t* n1, int64_t* n2) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        if (nf < 1 || !ntt_supported(F.p, nf))
            throw Error(ST_INVALID, "ntt: the prime has no 2-adic root for this length");
        ntt_shape(F.p, nf, n1, n2);
    });
}

int mmm_cu_ntt_phase_dev(int64_t p, int phase, const uint32_t* d_a, int64_t na,
                         const uint32_t* d_b, int64_t nb, int64_t start, int64_t n,
                         uint32_t* d_work_a, uint32_t* d_work_b, uint32_t* d_f, void* stream) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        if (na < 1 || nb < 1 || phase < 0 || phase > 2)
            throw Error(ST_INVALID, "ntt phase: bad operands or phase");
        if (!ntt_supported(F.p, na + nb - 1))
            throw Error(ST_INVALID, "ntt: the prime has no 2-adic root for this length");
        launch_ntt_phase(F, phase, d_a, na, d_b, nb, start, n, d_work_a, d_work_b, d_f,
                         as_stream(stream));
    });
}

int mmm_cu_divmod_fast(int64_t p, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb,
                       uint32_t* q, int64_t q_cap, int64_t* nq, uint32_t* r, int64_t r_cap,
                       int64_t* nr) {
    return guarded([&] {  // validation and results exactly as mmm_cu_divmod
        schedule_reset();
        const FieldParams F = field_or_throw(p);
        const char* wa = "division dividend";
        const char* wb = "division divisor";
        check_operand(a, na, wa);
        check_operand(b, nb, wb);
        const int64_t na0 = na;
        auto host_scan = [&] {  // the paths below that raise or return before the device
            check_canonical(a, na0, F.p, wa);
            check_canonical(b, nb, F.p, wb);
        };
        const bool scanned = na0 + nb <= DEV_CHECK_WORDS;
        if (scanned) host_scan();
        *nq = *nr = 0;
        try {
            if (nb == 0) throw Error(ST_DOMAIN, "divmod: division by the zero polynomial");
            na = trimmed_len(a, na);
            if (na < nb) {
                host_scan();
                need_cap(r_cap, na, "division remainder");
                if (na) std::memcpy(r, a, size_t(na) * 4);
                *nr = na;
                return;
            }
            if (b[nb - 1] == 0) throw Error(ST_DOMAIN, "field: inverse of zero");
            need_cap(q_cap, na - nb + 1, "division quotient");
            need_cap(r_cap, nb - 1, "division remainder");
        } catch (Error&) {
            host_scan();
            throw;
        }
        cudaStream_t st = thread_stream();
        checked_call(st, !scanned, F.p, a, na, wa, b, nb, wb,
                     [&](Scratch& sc, const uint32_t* da, const uint32_t* db) {
                         uint32_t* dq = sc.get<uint32_t>(size_t(na - nb + 1));
                         uint32_t* dr = sc.get<uint32_t>(size_t(nb));
                         launch_divmod_fast(F, da, na, db, nb, dq, dr, st);
                         to_host(q, dq, na - nb + 1, st);
                         to_host(r, dr, nb - 1, st);
                     });
        *nq = trimmed_len(q, na - nb + 1);
        *nr = trimmed_len(r, nb - 1);
    });
}

int mmm_cu_divmod_fast_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b,
                           int64_t nb, uint32_t* d_q, uint32_t* d_r, void* stream) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        if (nb < 1 || na < nb) throw Error(ST_INVALID, "division: requires deg a >= deg b >= 0");
        launch_divmod_fast(F, d_a, na, d_b, nb, d_q, d_r, as_stream(stream));
    });
}

int mmm_cu_divmod_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b, int64_t nb,
                      int64_t s, uint32_t* d_q, uint32_t* d_r, void* stream) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        if (nb < 1 || na < nb) throw Error(ST_INVALID, "division: requires deg a >= deg b >= 0");
        launch_divmod(F, d_a, na, d_b, nb, d_q, d_r, s, as_stream(stream));
    });
}

int mmm_cu_divmod_batched(int64_t p, const uint32_t* A, int64_t lda, int64_t na,
                          const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, int64_t s,
                          uint32_t* Q, int64_t ldq, uint32_t* R, int64_t ldr) {
    return guarded([&] {
        schedule_reset();
        const FieldParams F = field_or_throw(p);
        if (nb < 1 || na < nb || count < 0 || lda < na || ldb < nb || ldq < na - nb + 1 ||
            ldr < nb - 1)
            throw Error(ST_INVALID, "division batch: bad shape");
        for (int64_t i = 0; i < count; ++i)  // the divisors' leads: one word per row, on the host
            if (B[i * ldb + nb - 1] == 0) throw Error(ST_DOMAIN, "field: inverse of zero");
        if (count == 0) return;
        const int64_t lq = na - nb + 1, lr = nb - 1;
        pipelined_batch(F, count,
                        {{A, lda, na, "division batch dividend"},
                         {B, ldb, nb, "division batch divisor"}},
                        {{Q, ldq, lq}, {R, ldr, lr}},
                        [&](const std::vector<uint32_t*>& in, const std::vector<uint32_t*>& out,
                            int64_t c, cudaStream_t st) {
                            launch_divmod_batched(F, in[0], na, na, in[1], nb, nb, c, out[0], lq,
                                                  out[1], std::max<int64_t>(lr, 1), s, st);
                        });
    });
}

int mmm_cu_divmod_batched_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                              const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                              int64_t s, uint32_t* d_Q, int64_t ldq, uint32_t* d_R, int64_t ldr,
                              void* stream) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        if (nb < 1 || na < nb || count < 0 || lda < na || ldb < nb || ldq < na - nb + 1 ||
            ldr < nb - 1)
            throw Error(ST_INVALID, "division batch: bad shape");
        if (count)
            launch_divmod_batched(F, d_A, lda, na, d_B, ldb, nb, count, d_Q, ldq, d_R, ldr, s,
                                  as_stream(stream));
    });
}

// ---------------------------------------------------------------- gcd -----
int mmm_cu_gcd(int64_t p, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb, int64_t s,
               uint32_t* g, int64_t g_cap, int64_t* ng) {
    return guarded([&] {
        schedule_reset();
        const FieldParams F = field_or_throw(p);
        check_canonical(a, na, F.p, "gcd first operand");
        check_canonical(b, nb, F.p, "gcd second operand");
        na = trimmed_len(a, na);
        nb = trimmed_len(b, nb);
        *ng = 0;
        if (na == 0 && nb == 0) throw Error(ST_DOMAIN, "gcd: both inputs are zero");
        need_cap(g_cap, std::max(na, nb), "gcd");
        cudaStream_t st = thread_stream();
        int64_t len = 0;
        {
            Scratch sc(st);
            const uint32_t* da = to_device(sc, a, na);
            const uint32_t* db = to_device(sc, b, nb);
            uint32_t* dg = sc.get<uint32_t>(size_t(std::max(na, nb)));
            int64_t* dng = sc.get<int64_t>(1);
            launch_gcd(F, da, na, db, nb, dg, dng, s, st);
            // one synchronisation: the length and the whole result buffer come back
            // together into pinned staging, then len words go to the caller
            const int64_t n = std::max(na, nb);
            uint32_t* stage = pinned_stage(size_t(n) * 4 + 8);
            MMM_CUDA(cudaMemcpyAsync(stage, dng, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            MMM_CUDA(cudaMemcpyAsync(stage + 2, dg, size_t(n) * 4, cudaMemcpyDeviceToHost, st));
            sync(st);
            std::memcpy(&len, stage, sizeof(int64_t));
            if (len < 0 || len > n) throw Error(ST_SIM, "gcd: batch made no progress");
            std::memcpy(g, stage + 2, size_t(len) * 4);
        }
        *ng = len;
    });
}

int mmm_cu_gcd_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b, int64_t nb,
                   int64_t s, uint32_t* d_g, int64_t* d_ng, void* stream) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        if (na < 0 || nb < 0 || (na == 0 && nb == 0))
            throw Error(ST_DOMAIN, "gcd: both inputs are zero");
        launch_gcd(F, d_a, na, d_b, nb, d_g, d_ng, s, as_stream(stream));
    });
}

// ---------------------------------------------------------------- NTT -----
int mmm_cu_ntt_mul(int64_t p, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb,
                   uint32_t* f, int64_t f_cap, int64_t* nf) {
    return guarded([&] {
        schedule_reset();
        const FieldParams F = field_or_throw(p);
        const char* wa = "ntt first operand";
        const char* wb = "ntt second operand";
        check_operand(a, na, wa);
        check_operand(b, nb, wb);
        const int64_t na0 = na, nb0 = nb;
        auto host_scan = [&] {
            check_canonical(a, na0, F.p, wa);
            check_canonical(b, nb0, F.p, wb);
        };
        const bool scanned = na0 + nb0 <= DEV_CHECK_WORDS;
        if (scanned) host_scan();
        *nf = 0;
        na = trimmed_len(a, na);
        nb = trimmed_len(b, nb);
        if (na == 0 || nb == 0) {
            host_scan();
            return;
        }
        try {
            if (!ntt_supported(F.p, na + nb - 1))
                throw Error(ST_INVALID, "ntt: p has no 2-adic root of unity of the needed order");
            need_cap(f_cap, na + nb - 1, "ntt");
        } catch (Error&) {
            host_scan();
            throw;
        }
        cudaStream_t st = thread_stream();
        checked_call(st, !scanned, F.p, a, na, wa, b, nb, wb,
                     [&](Scratch& sc, const uint32_t* da, const uint32_t* db) {
                         uint32_t* df = sc.get<uint32_t>(size_t(na + nb - 1));
                         launch_ntt_mul(F, da, na, db, nb, df, st);
                         to_host(f, df, na + nb - 1, st);
                     });
        *nf = trimmed_len(f, na + nb - 1);
    });
}

int mmm_cu_ntt_mul_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b,
                       int64_t nb, uint32_t* d_f, void* stream) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        if (na < 1 || nb < 1) throw Error(ST_INVALID, "ntt: operands must be nonzero");
        if (!ntt_supported(F.p, na + nb - 1))
            throw Error(ST_INVALID, "ntt: p has no 2-adic root of unity of the needed order");
        launch_ntt_mul(F, d_a, na, d_b, nb, d_f, as_stream(stream));
    });
}

int mmm_cu_ntt_mul_batched(int64_t p, const uint32_t* A, int64_t lda, int64_t na,
                           const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, uint32_t* Fo,
                           int64_t ldf) {
    return guarded([&] {
        schedule_reset();
        const FieldParams F = field_or_throw(p);
        if (na < 1 || nb < 1 || count < 0 || lda < na || ldb < nb || ldf < na + nb - 1)
            throw Error(ST_INVALID, "ntt batch: bad shape");
        if (!ntt_supported(F.p, na + nb - 1))
            throw Error(ST_INVALID, "ntt: p has no 2-adic root of unity of the needed order");
        if (count == 0) return;
        const int64_t nf = na + nb - 1;
        pipelined_batch(F, count,
                        {{A, lda, na, "ntt batch first operand"},
                         {B, ldb, nb, "ntt batch second operand"}},
                        {{Fo, ldf, nf}},
                        [&](const std::vector<uint32_t*>& in, const std::vector<uint32_t*>& out,
                            int64_t c, cudaStream_t st) {
                            launch_ntt_mul_batched(F, in[0], na, na, in[1], nb, nb, c, out[0], nf, st);
                        });
    });
}

int mmm_cu_ntt_mul_batched_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                               const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                               uint32_t* d_F, int64_t ldf, void* stream) {
    return guarded([&] {
        const FieldParams F = field_or_throw(p);
        if (na < 1 || nb < 1 || count < 0 || lda < na || ldb < nb || ldf < na + nb - 1)
            throw Error(ST_INVALID, "ntt batch: bad shape");
        if (!ntt_supported(F.p, na + nb - 1))
            throw Error(ST_INVALID, "ntt: p has no 2-adic root of unity of the needed order");
        if (count)
            launch_ntt_mul_batched(F, d_A, lda, na, d_B, ldb, nb, count, d_F, ldf,
                                   as_stream(stream));
    });
}

}  // extern "C"
