// multi.cu -- one host process driving several GPUs through the C ABI
// (include/mmm_cu.h, "several devices"), without PyTorch or NCCL.
//
// Batched instances are independent (cfg4 batch, cfg5): the
// `count` instances split into contiguous, near-equal shares, one per entry
// of the device list.  Two flavours:
//
//  * host buffers (mmm_cu_*_batched_multi): one worker thread per share binds
//    its device and runs the single-device host entry point on its rows (H2D
//    of its share, kernel, D2H of its rows) -- all devices at once;
//  * device buffers on the root devices[0] (mmm_cu_*_batched_multi_dev): the
//    root's inputs are scattered over NVLink (peer copies into each device's
//    scratch), every device's kernel stores its rows straight into the root's
//    output through peer access (the fan-out epilogue: the gather is fused into
//    the producing kernel), and the root's stream waits on every device with
//    events.  Asynchronous on the root stream; nothing synchronises the host.
//
// A device may appear more than once (its shares run on separate streams):
// this is how the scatter/fused-gather logic is exercised on one GPU.
#include <cuda_runtime.h>

#include <condition_variable>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mmm_cu.h"
#include "common.cuh"

namespace mmm_cu {
namespace {

std::pair<int64_t, int64_t> share(int64_t count, int n, int r) {
    const int64_t base = count / n, extra = count % n;
    const int64_t lo = r * base + std::min<int64_t>(r, extra);
    return {lo, lo + base + (r < extra ? 1 : 0)};
}

std::vector<int> device_list(const int32_t* devices, int32_t n_dev) {
    if (devices == nullptr || n_dev < 1 || n_dev > MMM_MAX_FAN * 8)
        throw Error(ST_INVALID, "devices: need 1..64 device ordinals");
    int have = 0;
    MMM_CUDA(cudaGetDeviceCount(&have));
    std::vector<int> d(devices, devices + n_dev);
    for (int x : d)
        if (x < 0 || x >= have)
            throw Error(ST_INVALID, "devices: ordinal " + std::to_string(x) + " out of range");
    return d;
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int dev = 0;
    DeviceGuard() { cudaGetDevice(&dev); }
    ~DeviceGuard() { cudaSetDevice(dev); }
};

// ---- persistent workers: one host thread per (device, share slot) ---------
struct Worker {
    std::mutex m;
    std::condition_variable cv;
    std::deque<std::function<void()>> jobs;
    explicit Worker(int dev) {
        std::thread([this, dev] {
            cudaSetDevice(dev);
            for (;;) {
                std::function<void()> job;
                {
                    std::unique_lock<std::mutex> lk(m);
                    cv.wait(lk, [&] { return !jobs.empty(); });
                    job = std::move(jobs.front());
                    jobs.pop_front();
                }
                job();
            }
        }).detach();  // lives for the process (its thread state is per device)
    }
    void post(std::function<void()> f) {
        {
            std::lock_guard<std::mutex> lk(m);
            jobs.push_back(std::move(f));
        }
        cv.notify_one();
    }
};

Worker& worker(int dev, int slot) {
    static std::mutex mu;
    static auto* pool = new std::map<std::pair<int, int>, std::unique_ptr<Worker>>();
    std::lock_guard<std::mutex> lk(mu);
    auto& w = (*pool)[{dev, slot}];
    if (!w) w = std::make_unique<Worker>(dev);
    return *w;
}

// Runs fn(r) for every share on its worker; rethrows the first failure.
void run_shares(const std::vector<int>& devs, const std::function<int(int)>& fn) {
    struct Result {
        std::mutex m;
        std::condition_variable cv;
        int left;
        int status = 0;
        std::string msg;
    };
    auto res = std::make_shared<Result>();
    res->left = int(devs.size());
    for (int r = 0; r < int(devs.size()); ++r) {
        worker(devs[r], r).post([res, r, &fn] {
            const int st = fn(r);
            std::string msg = st ? mmm_last_error() : "";
            std::lock_guard<std::mutex> lk(res->m);
            if (st && !res->status) {
                res->status = st;
                res->msg = "share " + std::to_string(r) + ": " + msg;
            }
            if (--res->left == 0) res->cv.notify_all();
        });
    }
    std::unique_lock<std::mutex> lk(res->m);
    res->cv.wait(lk, [&] { return res->left == 0; });
    if (res->status) throw Error(res->status, res->msg);
}

// ---- device flavour: peer access, per-share streams and events ------------
void enable_peer(int dev, int root) {
    if (dev == root) return;
    static std::mutex mu;
    static std::set<std::pair<int, int>> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({dev, root})) return;
    int ok = 0;
    MMM_CUDA(cudaDeviceCanAccessPeer(&ok, dev, root));
    if (!ok)
        throw Error(ST_CUDA, "devices: no peer access from device " + std::to_string(dev) +
                                 " to device " + std::to_string(root));
    MMM_CUDA(cudaSetDevice(dev));
    const cudaError_t e = cudaDeviceEnablePeerAccess(root, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
    else
        MMM_CUDA(e);
    done.insert({dev, root});
}

// The calling thread's stream and event for share slot r on device dev.
struct Lane {
    cudaStream_t st = nullptr;
    cudaEvent_t done = nullptr;
};
Lane& lane(int dev, int r) {
    thread_local std::map<std::pair<int, int>, Lane> lanes;
    Lane& l = lanes[{dev, r}];
    if (!l.st) {
        MMM_CUDA(cudaSetDevice(dev));
        MMM_CUDA(cudaStreamCreateWithFlags(&l.st, cudaStreamNonBlocking));
        MMM_CUDA(cudaEventCreateWithFlags(&l.done, cudaEventDisableTiming));
    }
    return l;
}

cudaEvent_t fork_event(int root) {
    thread_local std::map<int, cudaEvent_t> evs;
    cudaEvent_t& e = evs[root];
    if (!e) {
        MMM_CUDA(cudaSetDevice(root));
        MMM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return e;
}

// Copies rows [lo, hi) of a root matrix (leading dimension ld, n words used
// per row) into dst on `dev` (same leading dimension), stream-ordered on st.
void scatter_rows(uint32_t* dst, int dev, const uint32_t* src, int root, int64_t rows, int64_t ld,
                  int64_t n, cudaStream_t st) {
    if (rows <= 0) return;
    const size_t bytes = size_t((rows - 1) * ld + n) * 4;
    if (dev == root)
        MMM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
    else
        MMM_CUDA(cudaMemcpyPeerAsync(dst, dev, src, root, bytes, st));
}

// One device-flavour batched call: `body(r, dev, lo, hi, st)` launches share
// r's work on `dev` (current) and stream st, reading its scattered inputs.
template <class Body>
void fork_join(const std::vector<int>& devs, int64_t count, cudaStream_t root_st, Body body) {
    const int root = devs[0];
    DeviceGuard guard;
    for (int d : devs) enable_peer(d, root);
    MMM_CUDA(cudaSetDevice(root));
    const cudaEvent_t fork = fork_event(root);
    MMM_CUDA(cudaEventRecord(fork, root_st));  // the root's inputs are ready
    const int n = int(devs.size());
    for (int r = 0; r < n; ++r) {
        const auto [lo, hi] = share(count, n, r);
        if (hi <= lo) continue;
        Lane& l = lane(devs[r], r);
        MMM_CUDA(cudaSetDevice(devs[r]));
        MMM_CUDA(cudaStreamWaitEvent(l.st, fork, 0));
        body(r, devs[r], lo, hi, l.st);
        MMM_CUDA(cudaEventRecord(l.done, l.st));
        MMM_CUDA(cudaSetDevice(root));
        MMM_CUDA(cudaStreamWaitEvent(root_st, l.done, 0));  // join
    }
}

}  // namespace
}  // namespace mmm_cu

using namespace mmm_cu;

extern "C" {

int mmm_cu_mul_batched_multi(int64_t p, const uint32_t* A, int64_t lda, int64_t na,
                             const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, int64_t s,
                             uint32_t* F, int64_t ldf, const int32_t* devices, int32_t n_dev) {
    return guarded([&] {
        const auto devs = device_list(devices, n_dev);
        if (count < 0) throw Error(ST_INVALID, "multiplication batch: bad shape");
        const int n = int(devs.size());
        run_shares(devs, [&](int r) {
            const auto [lo, hi] = share(count, n, r);
            return mmm_cu_mul_batched(p, A + lo * lda, lda, na, B + lo * ldb, ldb, nb, hi - lo, s,
                                      F + lo * ldf, ldf);
        });
    });
}

int mmm_cu_divmod_batched_multi(int64_t p, const uint32_t* A, int64_t lda, int64_t na,
                                const uint32_t* B, int64_t ldb, int64_t nb, int64_t count,
                                int64_t s, uint32_t* Q, int64_t ldq, uint32_t* R, int64_t ldr,
                                const int32_t* devices, int32_t n_dev) {
    return guarded([&] {
        const auto devs = device_list(devices, n_dev);
        if (count < 0) throw Error(ST_INVALID, "division batch: bad shape");
        const int n = int(devs.size());
        run_shares(devs, [&](int r) {
            const auto [lo, hi] = share(count, n, r);
            return mmm_cu_divmod_batched(p, A + lo * lda, lda, na, B + lo * ldb, ldb, nb, hi - lo,
                                         s, Q + lo * ldq, ldq, R + lo * ldr, ldr);
        });
    });
}

int mmm_cu_ntt_mul_batched_multi(int64_t p, const uint32_t* A, int64_t lda, int64_t na,
                                 const uint32_t* B, int64_t ldb, int64_t nb, int64_t count,
                                 uint32_t* F, int64_t ldf, const int32_t* devices, int32_t n_dev) {
    return guarded([&] {
        const auto devs = device_list(devices, n_dev);
        if (count < 0) throw Error(ST_INVALID, "ntt batch: bad shape");
        const int n = int(devs.size());
        run_shares(devs, [&](int r) {
            const auto [lo, hi] = share(count, n, r);
            return mmm_cu_ntt_mul_batched(p, A + lo * lda, lda, na, B + lo * ldb, ldb, nb, hi - lo,
                                          F + lo * ldf, ldf);
        });
    });
}

int mmm_cu_mul_batched_multi_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                                 const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                                 int64_t s, uint32_t* d_F, int64_t ldf, const int32_t* devices,
                                 int32_t n_dev, void* stream) {
    return guarded([&] {
        const FieldParams Fp = [&] {
            const int st = mmm_field_check(p);
            if (st) throw Error(st, mmm_last_error());
            return make_field(uint32_t(p));
        }();
        const auto devs = device_list(devices, n_dev);
        if (na < 1 || nb < 1 || count < 0 || lda < na || ldb < nb || ldf < na + nb - 1)
            throw Error(ST_INVALID, "multiplication batch: bad shape");
        if (count == 0) return;
        const int root = devs[0];
        fork_join(devs, count, static_cast<cudaStream_t>(stream),
                  [&](int, int dev, int64_t lo, int64_t hi, cudaStream_t st) {
                      Scratch sc(st);
                      const int64_t k = hi - lo;
                      uint32_t* a = sc.get<uint32_t>(size_t((k - 1) * lda + na));
                      uint32_t* b = sc.get<uint32_t>(size_t((k - 1) * ldb + nb));
                      scatter_rows(a, dev, d_A + lo * lda, root, k, lda, na, st);
                      scatter_rows(b, dev, d_B + lo * ldb, root, k, ldb, nb, st);
                      // rows land in the root's output over NVLink (fused gather)
                      launch_mul_batched_fan(Fp, a, lda, na, b, ldb, nb, k, fan_of(d_F + lo * ldf),
                                             ldf, s, st);
                  });
    });
}

int mmm_cu_divmod_batched_multi_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                                    const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                                    int64_t s, uint32_t* d_Q, int64_t ldq, uint32_t* d_R,
                                    int64_t ldr, const int32_t* devices, int32_t n_dev,
                                    void* stream) {
    return guarded([&] {
        const FieldParams Fp = [&] {
            const int st = mmm_field_check(p);
            if (st) throw Error(st, mmm_last_error());
            return make_field(uint32_t(p));
        }();
        const auto devs = device_list(devices, n_dev);
        if (nb < 1 || na < nb || count < 0 || lda < na || ldb < nb || ldq < na - nb + 1 ||
            ldr < nb - 1)
            throw Error(ST_INVALID, "division batch: bad shape");
        if (count == 0) return;
        const int root = devs[0];
        fork_join(devs, count, static_cast<cudaStream_t>(stream),
                  [&](int, int dev, int64_t lo, int64_t hi, cudaStream_t st) {
                      Scratch sc(st);
                      const int64_t k = hi - lo;
                      uint32_t* a = sc.get<uint32_t>(size_t((k - 1) * lda + na));
                      uint32_t* b = sc.get<uint32_t>(size_t((k - 1) * ldb + nb));
                      scatter_rows(a, dev, d_A + lo * lda, root, k, lda, na, st);
                      scatter_rows(b, dev, d_B + lo * ldb, root, k, ldb, nb, st);
                      launch_divmod_batched_fan(Fp, a, lda, na, b, ldb, nb, k,
                                                fan_of(d_Q + lo * ldq), ldq,
                                                fan_of(d_R + lo * ldr), ldr, s, st);
                  });
    });
}

int mmm_cu_ntt_mul_batched_multi_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                                     const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                                     uint32_t* d_F, int64_t ldf, const int32_t* devices,
                                     int32_t n_dev, void* stream) {
    return guarded([&] {
        const FieldParams Fp = [&] {
            const int st = mmm_field_check(p);
            if (st) throw Error(st, mmm_last_error());
            return make_field(uint32_t(p));
        }();
        const auto devs = device_list(devices, n_dev);
        if (na < 1 || nb < 1 || count < 0 || lda < na || ldb < nb || ldf < na + nb - 1)
            throw Error(ST_INVALID, "ntt batch: bad shape");
        if (!ntt_supported(Fp.p, na + nb - 1))
            throw Error(ST_INVALID, "ntt: p has no 2-adic root of unity of the needed order");
        if (count == 0) return;
        const int root = devs[0];
        const int64_t nf = na + nb - 1;
        fork_join(devs, count, static_cast<cudaStream_t>(stream),
                  [&](int, int dev, int64_t lo, int64_t hi, cudaStream_t st) {
                      Scratch sc(st);
                      const int64_t k = hi - lo;
                      uint32_t* a = sc.get<uint32_t>(size_t((k - 1) * lda + na));
                      uint32_t* b = sc.get<uint32_t>(size_t((k - 1) * ldb + nb));
                      uint32_t* f = sc.get<uint32_t>(size_t(k * nf));
                      scatter_rows(a, dev, d_A + lo * lda, root, k, lda, na, st);
                      scatter_rows(b, dev, d_B + lo * ldb, root, k, ldb, nb, st);
                      launch_ntt_mul_batched(Fp, a, lda, na, b, ldb, nb, k, f, nf, st);
                      // rows pushed into the root's output over NVLink (one copy
                      // per row block: the root's leading dimension may differ)
                      if (ldf == nf)
                          launch_fanout_copy(f, k * nf, fan_of(d_F + lo * ldf), st);
                      else
                          MMM_CUDA(cudaMemcpy2DAsync(d_F + lo * ldf, size_t(ldf) * 4, f,
                                                     size_t(nf) * 4, size_t(nf) * 4, size_t(k),
                                                     cudaMemcpyDefault, st));
                  });
    });
}

}  // extern "C"
