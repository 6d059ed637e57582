// mmm_b200.hpp -- C++ drop-in for the reference's arithmetic entry points
// (/root/reference/proj/include/mmm/*.hpp, namespace mmm), backed by the
// sm_100a kernels through the C ABI in mmm_cu.h.  A caller of the reference
// (mmm_cli.cpp do_run/do_verify, bench.cpp, the unit tests) recompiles against
// these declarations and links libmmm_b200.so instead of the simulator.
//
// Kept identical to the reference: names, argument meaning, Poly/Field
// semantics, exception types (std::invalid_argument, std::domain_error,
// SimError) and the capacity rules of the kernel programs (2l <= Z, 7s <= Z,
// 6s <= Z, 2sl+2s-1 <= Z, s >= 2 for the blocked GCD).
// Changed: SimReport keeps the reference's shape but is filled from the real
// launch schedule of the B200 run (simulator-only counters are zero); Rat is a
// Boost-free 64-bit rational with the subset of the API the callers use.
#pragma once

#include <cstdint>
#include <initializer_list>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace mmm {

// ----------------------------------------------------------- rational ----
class Rat {  // rational.hpp:12-62 stand-in (exact, 64-bit, normalised)
public:
    Rat(std::int64_t n = 0, std::int64_t d = 1);
    std::int64_t num() const { return n_; }
    std::int64_t den() const { return d_; }
    double to_double() const { return double(n_) / double(d_); }
    std::string str() const;
    friend Rat operator+(const Rat& a, const Rat& b);
    friend Rat operator-(const Rat& a, const Rat& b);
    friend Rat operator*(const Rat& a, const Rat& b);
    friend Rat operator/(const Rat& a, const Rat& b);
    friend bool operator==(const Rat& a, const Rat& b) { return a.n_ == b.n_ && a.d_ == b.d_; }
    friend bool operator!=(const Rat& a, const Rat& b) { return !(a == b); }
    friend bool operator<(const Rat& a, const Rat& b);
    friend bool operator<=(const Rat& a, const Rat& b) { return !(b < a); }
    friend bool operator>(const Rat& a, const Rat& b) { return b < a; }
    friend bool operator>=(const Rat& a, const Rat& b) { return !(a < b); }

private:
    std::int64_t n_, d_;
};

// -------------------------------------------------------------- field ----
class Field {  // field.hpp:9-39
public:
    explicit Field(std::int64_t p);  // std::invalid_argument unless prime, 2 <= p < 2^31
    std::int64_t p() const { return p_; }
    std::int64_t add(std::int64_t a, std::int64_t b) const { return a + b >= p_ ? a + b - p_ : a + b; }
    std::int64_t sub(std::int64_t a, std::int64_t b) const { return a - b < 0 ? a - b + p_ : a - b; }
    std::int64_t mul(std::int64_t a, std::int64_t b) const { return (a * b) % p_; }
    std::int64_t neg(std::int64_t a) const { return a == 0 ? 0 : p_ - a; }
    std::int64_t inv(std::int64_t a) const;  // std::domain_error on 0
    std::int64_t divide(std::int64_t a, std::int64_t b) const { return mul(a, inv(b)); }
    std::int64_t reduce(std::int64_t x) const {
        const std::int64_t r = x % p_;
        return r < 0 ? r + p_ : r;
    }

private:
    std::int64_t p_;
};

// --------------------------------------------------------------- poly ----
struct Poly {  // poly.hpp:16-30: ascending, trimmed, zero = empty
    std::vector<std::int64_t> c;
    Poly() = default;
    explicit Poly(std::vector<std::int64_t> coeffs) : c(std::move(coeffs)) {}
    Poly(std::initializer_list<std::int64_t> coeffs) : c(coeffs) {}
    bool is_zero() const { return c.empty(); }
    std::int64_t degree() const { return std::int64_t(c.size()) - 1; }
    std::int64_t lead() const { return c.back(); }
    friend bool operator==(const Poly& a, const Poly& b) { return a.c == b.c; }
    friend bool operator!=(const Poly& a, const Poly& b) { return a.c != b.c; }
};

Poly trimmed(Poly p);
Poly monic(const Poly& p, const Field& F);
Poly random_poly(std::mt19937_64& rng, std::int64_t terms, const Field& F);
std::string to_string(const Poly& p);

// --------------------------------------- oracle-style entry points (GPU) --
Poly oracle_mul(const Poly& a, const Poly& b, const Field& F);      // oracle.hpp:14
Poly oracle_mul_alt(const Poly& a, const Poly& b, const Field& F);  // oracle.hpp:18 (NTT when p allows)
Poly oracle_add(const Poly& a, const Poly& b, const Field& F);
Poly oracle_sub(const Poly& a, const Poly& b, const Field& F);
std::pair<Poly, Poly> oracle_divmod(const Poly& a, const Poly& b, const Field& F);  // oracle.hpp:25
Poly oracle_gcd(const Poly& a, const Poly& b, const Field& F);                      // oracle.hpp:29

// --------------------------------------------- kernel-program entry points --
enum class Variant { naive, optimized };  // variant.hpp:18

struct SimError : std::runtime_error {  // machine.hpp:20-22
    using std::runtime_error::runtime_error;
};

struct MachineParams {  // machine.hpp:24-28
    Rat U = Rat(2);
    std::int64_t Z = 1024;
    bool parallel = true;
};

// ---- metrics (metrics.hpp:12-72, simtypes.hpp:16-20), same shape ---------
// Filled from the launch schedule the B200 actually ran (mmm_cu_last_schedule):
// one KernelMetrics per CUDA launch (name, blocks, threads per block), and the
// structural metrics of that launch DAG -- a chain on one stream, so
// N = sum of blocks, L = pi = launches, K = max blocks (graph.cpp:56-110).
// The per-thread work/span/overhead counters (W, S, O, C, alpha, beta,
// max_accesses, per_block) exist only in the reference's simulator; here they
// are 0 / empty.  device_ms and block_param are B200 additions.
struct BlockMetrics {  // metrics.hpp:22-31
    std::int64_t W = 0, S = 0, alpha = 0, beta = 0, max_accesses = 0;
    Rat O;
    Rat C() const { return Rat(S) + O; }
};
struct KernelMetrics {  // metrics.hpp:36-48
    std::string name;
    std::int64_t blocks = 0;
    std::int64_t threads = 0;  // threads per block
    std::vector<BlockMetrics> per_block;
    std::int64_t W() const { return 0; }
    std::int64_t S() const { return 0; }
    Rat O() const { return Rat(0); }
    Rat max_block_C() const { return Rat(0); }
    std::int64_t max_accesses() const { return 0; }
};
struct StructuralMetrics {  // metrics.hpp:51-56
    std::int64_t N = 0;   // total blocks over all kernels
    std::int64_t L = 0;   // vertices on a longest path
    std::int64_t K = 0;   // maximum antichain weight (blocks)
    std::int64_t pi = 0;  // minimum number of parallel rounds (= L)
};
struct ProgramMetrics {  // metrics.hpp:59-65
    std::int64_t W = 0;
    std::int64_t S = 0;
    Rat O;
    Rat C;
    StructuralMetrics structure;
};
struct SimReport {  // simtypes.hpp:16-20
    ProgramMetrics metrics;
    std::vector<KernelMetrics> kernels;
    std::int64_t max_thread_accesses = 0;
    // B200 additions
    std::int64_t block_param = 0;  // s (or l) the kernels used
    double device_ms = 0;          // wall time of the synchronous call
};

struct MulResult {  // multiplication.hpp:12-15
    Poly f;
    SimReport sim;
};
struct DivisionResult {  // division.hpp:7-11
    Poly q, r;
    SimReport sim;
};
struct GcdResult {  // gcd.hpp:7-10
    Poly g;
    SimReport sim;
};

MulResult run_multiplication(const MachineParams& mp, const Field& F, const Poly& a, const Poly& b,
                             std::int64_t s, std::int64_t l);
DivisionResult run_division(Variant variant, const MachineParams& mp, const Field& F,
                            const Poly& a, const Poly& b, std::int64_t block_param);
GcdResult run_gcd(Variant variant, const MachineParams& mp, const Field& F, const Poly& a,
                  const Poly& b, std::int64_t block_param);

namespace testhooks {
extern bool corrupt_division_output;  // testhooks.hpp:8 (mutation smoke test)
}

}  // namespace mmm
