/*
 * mmm_cu.h -- C ABI of the B200 (sm_100a) polynomial-arithmetic hot path.
 *
 * Drop-in boundary for the reference's arithmetic entry points
 * (/root/reference/proj/include/mmm/, namespace mmm):
 *
 *   mmm_cu_mul      <- Poly oracle_mul(const Poly&, const Poly&, const Field&)      oracle.hpp:14
 *                      MulResult run_multiplication(mp, F, a, b, s, l)             multiplication.hpp:29
 *   mmm_cu_divmod   <- pair<Poly,Poly> oracle_divmod(a, b, F)                       oracle.hpp:25
 *                      DivisionResult run_division(variant, mp, F, a, b, s)         division.hpp:18
 *   mmm_cu_gcd      <- Poly oracle_gcd(a, b, F)                                     oracle.hpp:29
 *                      GcdResult run_gcd(variant, mp, F, a, b, s)                   gcd.hpp:19
 *   mmm_cu_ntt_mul  <- (no reference symbol: FFT product is new scope, SURVEY §0;
 *                      its result is the unique product, == oracle_mul)
 *   mmm_field_check <- Field::Field(int64) validation                               field.cpp:20-25
 *   mmm_random_poly <- Poly random_poly(std::mt19937_64&, int64 terms, const Field&) poly.hpp:40
 *
 * Conventions (mirroring mmm::Poly, poly.hpp:16-30): a polynomial is a pointer
 * to ascending uint32 coefficients and a length; length 0 is the zero
 * polynomial.  Coefficients must be canonical residues in [0, p) of a prime
 * p with 2 <= p < 2^31.  Host-buffer entry points return TRIMMED results
 * (no leading zero words) with the length in *n_out, exactly like the
 * reference's Poly results; batched and device entry points write fixed,
 * untrimmed lengths.
 *
 * Errors: every entry point returns an mmm_status; the message of the last
 * failure on the calling thread is mmm_last_error().  MMM_INVALID_ARGUMENT
 * maps to std::invalid_argument (non-prime p, non-canonical coefficients,
 * output capacity), MMM_DOMAIN_ERROR to std::domain_error (division by the
 * zero polynomial, gcd of two zeros, inverse of zero), as the oracle throws
 * them (oracle.cpp:52,71; field.cpp:28).
 *
 * Threading: pure functions without global state; host entry points run on the
 * calling thread's CUDA stream of the current device (one per thread and
 * device) and are safe to call concurrently.  Device entry points are asynchronous on the
 * caller's stream (a cudaStream_t passed as void*; NULL = legacy default).
 */
#ifndef MMM_CU_H
#define MMM_CU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum mmm_status {
    MMM_OK = 0,
    MMM_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    MMM_DOMAIN_ERROR = 2,     /* std::domain_error */
    MMM_CUDA_ERROR = 3,
    MMM_NCCL_ERROR = 4,
    MMM_SIM_ERROR = 5 /* mmm::SimError (machine.hpp:20-22): internal invariant */
} mmm_status;

const char* mmm_last_error(void);
int mmm_version(void);
/* Number of CUDA kernels this library has launched in this process. */
uint64_t mmm_cu_launch_count(void);
/* The kernels the calling thread's last host-buffer compute call launched, in
 * launch order (all on one stream, so the launch DAG is a chain): name, grid
 * blocks and threads per block.  At most `cap` records are copied; *n gets
 * the total.  The drop-in's SimReport (include/mmm_b200.hpp) is built from
 * this: N = sum of blocks, L = pi = launches, K = max blocks
 * (graph.cpp:56-110 on a chain). */
typedef struct mmm_kernel_rec {
    char name[40];
    int64_t blocks;
    int32_t threads;
} mmm_kernel_rec;
int mmm_cu_last_schedule(mmm_kernel_rec* out, int32_t cap, int32_t* n);
/* Frees the calling thread's per-device streams, scratch arenas, zero buffers
 * and pinned staging (waiting for their queued work first).  They are also
 * freed when the thread exits; the next call recreates them. */
int mmm_cu_release_scratch(void);
/* mmm_cu_release_scratch() plus the process-wide NTT plans, after
 * synchronising every device.  No other thread may have calls in flight. */
int mmm_cu_release_all(void);

/* Page-locked host memory for results (process-wide pool): a buffer handed
 * back with mmm_cu_host_free() is kept and reused by the next request of the
 * same rounded size, so a caller that allocates its batched results this way
 * gets full-speed device-to-host copies without paying for page-locking on
 * every call.  Up to 2 GB of freed buffers are kept; mmm_cu_release_all()
 * returns them to the system. */
int mmm_cu_host_alloc(size_t bytes, void** out);
int mmm_cu_host_free(void* p);

/* ---- field and inputs (host) ------------------------------------------- */
int mmm_field_check(int64_t p);
/* a^-1 mod p in *out; MMM_DOMAIN_ERROR for a == 0 (Field::inv, field.cpp:27-42). */
int mmm_field_inv(int64_t a, int64_t p, int64_t* out);

typedef struct mmm_rng mmm_rng; /* std::mt19937_64 */
mmm_rng* mmm_rng_create(uint64_t seed);
void mmm_rng_destroy(mmm_rng* g);
uint64_t mmm_rng_next(mmm_rng* g);
/* random_poly (poly.cpp:20-29): `terms` coefficients uniform in [0, p),
 * leading one uniform in [1, p); same draws as the reference. */
int mmm_random_poly(mmm_rng* g, int64_t terms, int64_t p, uint32_t* out);

/* ---- host-buffer entry points (synchronous, trimmed results) ------------ */
/* f = a*b; f_cap >= na+nb-1.  s >= 1: the paper's program parameter (per-thread
 * register tile of the CUDA-core kernel); s <= 0: auto (large products run on
 * the integer tensor core).  l = threads-per-block hint (ignored on B200). */
int mmm_cu_mul(int64_t p, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb, int64_t s,
               int64_t l, uint32_t* f, int64_t f_cap, int64_t* nf);
/* (q, r) = divmod(a, b); q_cap >= na-nb+1, r_cap >= nb-1 (when na >= nb),
 * else q = 0 and r = trimmed a (r_cap >= na).  s = heads retired per step. */
int mmm_cu_divmod(int64_t p, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb,
                  int64_t s, uint32_t* q, int64_t q_cap, int64_t* nq, uint32_t* r, int64_t r_cap,
                  int64_t* nr);
/* The same (q, r), contract and errors as mmm_cu_divmod, in O(M(n)): Newton
 * inverse of rev(b) and NTT products (schoolbook products where the prime
 * lacks 2-adic roots).  No reference symbol: SURVEY §8f item 4. */
int mmm_cu_divmod_fast(int64_t p, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb,
                       uint32_t* q, int64_t q_cap, int64_t* nq, uint32_t* r, int64_t r_cap,
                       int64_t* nr);
/* g = monic gcd(a, b); g_cap >= max(na, nb).  s = steps per matrix batch. */
int mmm_cu_gcd(int64_t p, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb, int64_t s,
               uint32_t* g, int64_t g_cap, int64_t* ng);
/* f = a*b through a Stockham NTT; needs p - 1 divisible by the transform
 * length (next power of two >= na+nb-1), else MMM_INVALID_ARGUMENT. */
int mmm_cu_ntt_mul(int64_t p, const uint32_t* a, int64_t na, const uint32_t* b, int64_t nb,
                   uint32_t* f, int64_t f_cap, int64_t* nf);

/* ---- batched host entry points: `count` equal-shape instances, row-major
 *      with leading dimensions; outputs untrimmed (fixed lengths).  s <= 0 =
 *      auto: products of <= 4096-term operands and divisions of <= 8192 by
 *      <= 4096 terms run on the integer tensor core when the batch is large;
 *      s >= 1 selects the s-parameterised CUDA-core kernels. -------------- */
int mmm_cu_mul_batched(int64_t p, const uint32_t* A, int64_t lda, int64_t na, const uint32_t* B,
                       int64_t ldb, int64_t nb, int64_t count, int64_t s, uint32_t* F, int64_t ldf);
/* every B row must have a nonzero word at index nb-1; na >= nb.
 * Q rows hold na-nb+1 words, R rows nb-1 words. */
int mmm_cu_divmod_batched(int64_t p, const uint32_t* A, int64_t lda, int64_t na,
                          const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, int64_t s,
                          uint32_t* Q, int64_t ldq, uint32_t* R, int64_t ldr);
int mmm_cu_ntt_mul_batched(int64_t p, const uint32_t* A, int64_t lda, int64_t na,
                           const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, uint32_t* F,
                           int64_t ldf);

/* ---- device-pointer entry points (asynchronous on `stream`) -------------
 * Inputs: canonical, na, nb >= 1, leading words as for the host versions.
 * Outputs: fixed lengths (f: na+nb-1; q: na-nb+1; r: nb-1), untrimmed. */
int mmm_cu_mul_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b, int64_t nb,
                   int64_t s, uint32_t* d_f, void* stream);
int mmm_cu_divmod_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b, int64_t nb,
                      int64_t s, uint32_t* d_q, uint32_t* d_r, void* stream);
/* Sharded four-step NTT product (no reference symbol: SURVEY §8f item 4).
 * mmm_cu_ntt_shape: the transform for nf = na+nb-1 outputs is N = n1 x n2.
 * mmm_cu_ntt_phase_dev: phase 0 = forward column transforms [start, start+n)
 * of both operands into the N-word workspaces (layout w[n2*k1 + col]);
 * 1 = rows [start, start+n): forward, pointwise product, inverse (result in
 * d_work_a); 2 = inverse columns [start, start+n) into d_f (nf words, only
 * the positions of those columns).  Column slices are multiples of 4.  Ranks
 * exchange workspace blocks between phases (paper_1402_0264_b200/shard.py). */
int mmm_cu_ntt_shape(int64_t p, int64_t nf, int64_t* n1, int64_t* n2);
int mmm_cu_ntt_phase_dev(int64_t p, int phase, const uint32_t* d_a, int64_t na,
                         const uint32_t* d_b, int64_t nb, int64_t start, int64_t n,
                         uint32_t* d_work_a, uint32_t* d_work_b, uint32_t* d_f, void* stream);
int mmm_cu_divmod_fast_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b,
                           int64_t nb, uint32_t* d_q, uint32_t* d_r, void* stream);
/* Coefficients [k0, k1) of the product into d_f[0, k1 - k0): one rank's slice of
 * an output-range-sharded product (no reference symbol: B200 sharding). */
int mmm_cu_mul_range_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b,
                         int64_t nb, int64_t k0, int64_t k1, int64_t s, uint32_t* d_f,
                         void* stream);
/* d_g capacity max(na, nb); *d_ng (device int64) receives the gcd length. */
int mmm_cu_gcd_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b, int64_t nb,
                   int64_t s, uint32_t* d_g, int64_t* d_ng, void* stream);
int mmm_cu_ntt_mul_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b,
                       int64_t nb, uint32_t* d_f, void* stream);
int mmm_cu_mul_batched_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                           const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count, int64_t s,
                           uint32_t* d_F, int64_t ldf, void* stream);
int mmm_cu_divmod_batched_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                              const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                              int64_t s, uint32_t* d_Q, int64_t ldq, uint32_t* d_R, int64_t ldr,
                              void* stream);
int mmm_cu_ntt_mul_batched_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                               const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                               uint32_t* d_F, int64_t ldf, void* stream);

/* Fan-out variants of the sharded entry points.  `d_f` / `d_F` /
 * `d_Q` / `d_R` are HOST arrays of n_out (1..8) device pointers with the same
 * layout as the single-output call; every output word is stored into each of
 * them.  Passing the buffers of every rank (symmetric / IPC-mapped memory, peer
 * access over NVLink) fuses the all-gather of a sharded product or batch into
 * the producing kernel's epilogue: rank r's slice or rows land in every rank's
 * full result with no gather collective.  The caller orders the ranks after the
 * kernels (a barrier) before reading.  Reference interface replaced: the gather
 * of results the reference's callers do after run_multiplication / run_division
 * (bench.cpp:43-64, mmm_cli.cpp:207-221), which have no multi-GPU counterpart. */
int mmm_cu_mul_range_fanout_dev(int64_t p, const uint32_t* d_a, int64_t na, const uint32_t* d_b,
                                int64_t nb, int64_t k0, int64_t k1, int64_t s,
                                uint32_t* const* d_f, int32_t n_out, void* stream);
int mmm_cu_mul_batched_fanout_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                                  const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                                  int64_t s, uint32_t* const* d_F, int32_t n_out, int64_t ldf,
                                  void* stream);
/* Push n words of d_src into every one of the n_out (1..8) buffers d_dst[q]:
 * the gather for results whose kernels have no fan-out epilogue (the NTT
 * batch), as one peer-store kernel over NVLink instead of a collective. */
int mmm_cu_fanout_copy_dev(const uint32_t* d_src, int64_t n, uint32_t* const* d_dst,
                           int32_t n_out, void* stream);
int mmm_cu_divmod_batched_fanout_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                                     const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                                     int64_t s, uint32_t* const* d_Q, int64_t ldq,
                                     uint32_t* const* d_R, int64_t ldr, int32_t n_out,
                                     void* stream);

/* ---- one process, several GPUs (no PyTorch, no NCCL) ---------
 * `devices` lists n_dev device ordinals; the `count` independent instances are
 * split into contiguous near-equal shares, share r on devices[r] (a device may
 * repeat: its shares then run on separate streams).
 *
 * Host-buffer versions: one worker thread per share runs the single-device
 * host entry point on its rows (H2D of its share, kernels, D2H of its rows),
 * all devices concurrently; synchronous, same validation and errors as the
 * single-device calls (a failing share's status and message are returned). */
int mmm_cu_mul_batched_multi(int64_t p, const uint32_t* A, int64_t lda, int64_t na,
                             const uint32_t* B, int64_t ldb, int64_t nb, int64_t count, int64_t s,
                             uint32_t* F, int64_t ldf, const int32_t* devices, int32_t n_dev);
int mmm_cu_divmod_batched_multi(int64_t p, const uint32_t* A, int64_t lda, int64_t na,
                                const uint32_t* B, int64_t ldb, int64_t nb, int64_t count,
                                int64_t s, uint32_t* Q, int64_t ldq, uint32_t* R, int64_t ldr,
                                const int32_t* devices, int32_t n_dev);
int mmm_cu_ntt_mul_batched_multi(int64_t p, const uint32_t* A, int64_t lda, int64_t na,
                                 const uint32_t* B, int64_t ldb, int64_t nb, int64_t count,
                                 uint32_t* F, int64_t ldf, const int32_t* devices, int32_t n_dev);
/* Device-buffer versions: inputs and outputs live on the root devices[0] and
 * `stream` is a stream of the root.  Each share's inputs are copied from the
 * root over NVLink (peer copies), its kernel stores its rows straight into the
 * root's outputs through peer access (fan-out epilogue: the gather is fused
 * into the producing kernel; the NTT batch pushes its rows with one copy), and
 * `stream` waits on every device (events).  Asynchronous on `stream`.  Peer
 * access is enabled on first use; MMM_CUDA_ERROR if a device cannot reach the
 * root. */
int mmm_cu_mul_batched_multi_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                                 const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                                 int64_t s, uint32_t* d_F, int64_t ldf, const int32_t* devices,
                                 int32_t n_dev, void* stream);
int mmm_cu_divmod_batched_multi_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                                    const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                                    int64_t s, uint32_t* d_Q, int64_t ldq, uint32_t* d_R,
                                    int64_t ldr, const int32_t* devices, int32_t n_dev,
                                    void* stream);
int mmm_cu_ntt_mul_batched_multi_dev(int64_t p, const uint32_t* d_A, int64_t lda, int64_t na,
                                     const uint32_t* d_B, int64_t ldb, int64_t nb, int64_t count,
                                     uint32_t* d_F, int64_t ldf, const int32_t* devices,
                                     int32_t n_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MMM_CU_H */
