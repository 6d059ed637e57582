// mmm_b200.cpp -- the C++ drop-in (include/mmm_b200.hpp) over the C ABI.
//
// Every arithmetic entry point converts Poly <-> uint32 residues, calls the
// sm_100a library (mmm_cu_*), and rethrows its status as the exception the
// reference throws.  Input checks of the kernel programs follow
// proj/src/multiplication.cpp:25-34, division.cpp:182-196, gcd.cpp:340-357.
#include "../../include/mmm_b200.hpp"

#include <algorithm>
#include <chrono>
#include <numeric>
#include <vector>

#include "../../include/mmm_cu.h"

namespace mmm {

namespace testhooks {
bool corrupt_division_output = false;
}

namespace {

[[noreturn]] void rethrow(int st) {
    const std::string msg = mmm_last_error();
    if (st == MMM_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (st == MMM_DOMAIN_ERROR) throw std::domain_error(msg);
    if (st == MMM_SIM_ERROR) throw SimError(msg);
    throw std::runtime_error("CUDA: " + msg);
}
void ok(int st) {
    if (st != MMM_OK) rethrow(st);
}

std::vector<uint32_t> to_u32(const Poly& p) {
    std::vector<uint32_t> v(p.c.size());
    for (size_t i = 0; i < v.size(); ++i) {
        if (p.c[i] < 0 || p.c[i] > 0xFFFFFFFFll)
            throw std::invalid_argument("coefficients must be canonical field elements");
        v[i] = uint32_t(p.c[i]);
    }
    return v;
}
Poly from_u32(const uint32_t* w, int64_t n) {
    Poly out;
    out.c.assign(w, w + n);
    return out;
}

struct Clock {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    SimReport report(std::int64_t s) const {
        SimReport r;
        r.block_param = s;
        r.device_ms = std::chrono::duration<double, std::milli>(
                          std::chrono::steady_clock::now() - t0)
                          .count();
        int32_t n = 0;
        ok(mmm_cu_last_schedule(nullptr, 0, &n));
        std::vector<mmm_kernel_rec> recs(size_t(std::max(n, 0)));
        ok(mmm_cu_last_schedule(recs.data(), int32_t(recs.size()), &n));
        StructuralMetrics& st = r.metrics.structure;
        for (const auto& k : recs) {
            KernelMetrics km;
            km.name = k.name;
            km.blocks = k.blocks;
            km.threads = k.threads;
            st.N += k.blocks;
            st.K = std::max(st.K, k.blocks);
            r.kernels.push_back(std::move(km));
        }
        st.L = st.pi = std::int64_t(recs.size());
        return r;
    }
};

void canonical(const Poly& p, const Field& F, const char* who) {  // run_util.hpp:24-29
    for (std::int64_t c : p.c)
        if (c < 0 || c >= F.p())
            throw std::invalid_argument(std::string(who) +
                                        ": coefficients must be canonical field elements");
}

Poly gpu_mul(const Poly& a, const Poly& b, const Field& F, std::int64_t s, std::int64_t l) {
    if (a.is_zero() || b.is_zero()) return Poly{};
    const auto ua = to_u32(a), ub = to_u32(b);
    std::vector<uint32_t> f(ua.size() + ub.size() - 1);
    int64_t nf = 0;
    ok(mmm_cu_mul(F.p(), ua.data(), int64_t(ua.size()), ub.data(), int64_t(ub.size()), s, l,
                  f.data(), int64_t(f.size()), &nf));
    return from_u32(f.data(), nf);
}

std::pair<Poly, Poly> gpu_divmod(const Poly& a, const Poly& b, const Field& F, std::int64_t s) {
    const auto ua = to_u32(a), ub = to_u32(b);
    std::vector<uint32_t> q(std::max<size_t>(ua.size(), 1)), r(std::max<size_t>(ua.size(), 1));
    int64_t nq = 0, nr = 0;
    ok(mmm_cu_divmod(F.p(), ua.data(), int64_t(ua.size()), ub.data(), int64_t(ub.size()), s,
                     q.data(), int64_t(q.size()), &nq, r.data(), int64_t(r.size()), &nr));
    return {from_u32(q.data(), nq), from_u32(r.data(), nr)};
}

Poly gpu_gcd(const Poly& a, const Poly& b, const Field& F, std::int64_t s) {
    const auto ua = to_u32(a), ub = to_u32(b);
    std::vector<uint32_t> g(std::max<size_t>(std::max(ua.size(), ub.size()), 1));
    int64_t ng = 0;
    ok(mmm_cu_gcd(F.p(), ua.data(), int64_t(ua.size()), ub.data(), int64_t(ub.size()), s,
                  g.data(), int64_t(g.size()), &ng));
    return from_u32(g.data(), ng);
}

std::int64_t igcd(std::int64_t a, std::int64_t b) { return std::gcd(a < 0 ? -a : a, b < 0 ? -b : b); }

}  // namespace

// ----------------------------------------------------------------- Rat ----
Rat::Rat(std::int64_t n, std::int64_t d) : n_(n), d_(d) {
    if (d_ == 0) throw std::domain_error("Rat: zero denominator");
    if (d_ < 0) {
        n_ = -n_;
        d_ = -d_;
    }
    const std::int64_t g = igcd(n_, d_);
    if (g > 1) {
        n_ /= g;
        d_ /= g;
    }
}
std::string Rat::str() const {
    return d_ == 1 ? std::to_string(n_) : std::to_string(n_) + "/" + std::to_string(d_);
}
Rat operator+(const Rat& a, const Rat& b) { return Rat(a.n_ * b.d_ + b.n_ * a.d_, a.d_ * b.d_); }
Rat operator-(const Rat& a, const Rat& b) { return Rat(a.n_ * b.d_ - b.n_ * a.d_, a.d_ * b.d_); }
Rat operator*(const Rat& a, const Rat& b) { return Rat(a.n_ * b.n_, a.d_ * b.d_); }
Rat operator/(const Rat& a, const Rat& b) { return Rat(a.n_ * b.d_, a.d_ * b.n_); }
bool operator<(const Rat& a, const Rat& b) { return a.n_ * b.d_ < b.n_ * a.d_; }

// --------------------------------------------------------------- Field ----
Field::Field(std::int64_t p) : p_(p) {
    const int st = mmm_field_check(p);
    if (st != MMM_OK) throw std::invalid_argument(mmm_last_error());
}

std::int64_t Field::inv(std::int64_t a) const {
    int64_t out = 0;
    const int st = mmm_field_inv(a, p_, &out);
    if (st != MMM_OK) rethrow(st);
    return out;
}

// ---------------------------------------------------------------- Poly ----
Poly trimmed(Poly p) {
    auto it = std::find_if(p.c.rbegin(), p.c.rend(), [](std::int64_t v) { return v != 0; });
    p.c.erase(it.base(), p.c.end());
    return p;
}

Poly monic(const Poly& p, const Field& F) {
    if (p.is_zero()) return p;
    const std::int64_t s = F.inv(p.lead());
    Poly out = p;
    std::transform(out.c.begin(), out.c.end(), out.c.begin(),
                   [&](std::int64_t v) { return F.mul(v, s); });
    return out;
}

Poly random_poly(std::mt19937_64& rng, std::int64_t terms, const Field& F) {
    if (terms < 1) throw std::invalid_argument("random_poly: terms must be >= 1");
    std::uniform_int_distribution<std::int64_t> body(0, F.p() - 1), head(1, F.p() - 1);
    Poly out;
    out.c.reserve(size_t(terms));
    while (std::int64_t(out.c.size()) + 1 < terms) out.c.push_back(body(rng));
    out.c.push_back(head(rng));
    return out;
}

std::string to_string(const Poly& p) {
    std::string s;
    for (std::int64_t i = p.degree(); i >= 0; --i) {
        const std::int64_t v = p.c[size_t(i)];
        if (v == 0) continue;
        std::string term = (v != 1 || i == 0) ? std::to_string(v) : "";
        if (i > 0) term += (term.empty() ? "" : "*") + std::string(i == 1 ? "X" : "X^" + std::to_string(i));
        s += (s.empty() ? "" : " + ") + term;
    }
    return s.empty() ? "0" : s;
}

// -------------------------------------------------------- oracle-style ----
Poly oracle_mul(const Poly& a, const Poly& b, const Field& F) { return gpu_mul(a, b, F, 0, 128); }  // auto

Poly oracle_mul_alt(const Poly& a, const Poly& b, const Field& F) {
    if (a.is_zero() || b.is_zero()) return Poly{};
    const auto ua = to_u32(a), ub = to_u32(b);
    std::vector<uint32_t> f(ua.size() + ub.size() - 1);
    int64_t nf = 0;
    const int st = mmm_cu_ntt_mul(F.p(), ua.data(), int64_t(ua.size()), ub.data(),
                                  int64_t(ub.size()), f.data(), int64_t(f.size()), &nf);
    if (st == MMM_INVALID_ARGUMENT) return gpu_mul(a, b, F, 4, 128);  // p has no NTT roots
    ok(st);
    return from_u32(f.data(), nf);
}

static Poly addsub(const Poly& a, const Poly& b, const Field& F, bool sub) {
    Poly out;
    out.c.resize(std::max(a.c.size(), b.c.size()));
    for (size_t i = 0; i < out.c.size(); ++i) {
        const std::int64_t x = i < a.c.size() ? a.c[i] : 0, y = i < b.c.size() ? b.c[i] : 0;
        out.c[i] = sub ? F.sub(x, y) : F.add(x, y);
    }
    return trimmed(std::move(out));
}
Poly oracle_add(const Poly& a, const Poly& b, const Field& F) { return addsub(a, b, F, false); }
Poly oracle_sub(const Poly& a, const Poly& b, const Field& F) { return addsub(a, b, F, true); }

std::pair<Poly, Poly> oracle_divmod(const Poly& a, const Poly& b, const Field& F) {
    return gpu_divmod(a, b, F, 64);
}

Poly oracle_gcd(const Poly& a, const Poly& b, const Field& F) { return gpu_gcd(a, b, F, 64); }

// ------------------------------------------------------ kernel programs ----
MulResult run_multiplication(const MachineParams& mp, const Field& F, const Poly& a_in,
                             const Poly& b_in, std::int64_t s, std::int64_t l) {
    const Poly a = trimmed(a_in), b = trimmed(b_in);
    if (a.is_zero() || b.is_zero())
        throw std::invalid_argument("multiplication: operands must be nonzero");
    if (s < 1) throw std::invalid_argument("multiplication: s must be >= 1");
    if (l < 1) throw std::invalid_argument("multiplication: l must be >= 1");
    if (2 * s * l + 2 * s - 1 > mp.Z)
        throw std::invalid_argument("multiplication: requires 2*s*l + 2*s - 1 <= Z");
    canonical(a, F, "multiplication first operand");
    canonical(b, F, "multiplication second operand");
    Clock clk;
    MulResult res;
    res.f = gpu_mul(a, b, F, s, l);
    res.sim = clk.report(s);
    return res;
}

DivisionResult run_division(Variant variant, const MachineParams& mp, const Field& F,
                            const Poly& a_in, const Poly& b_in, std::int64_t block_param) {
    const Poly a = trimmed(a_in), b = trimmed(b_in);
    if (b.is_zero()) throw std::invalid_argument("division: divisor must be nonzero");
    if (a.is_zero() || a.degree() < b.degree())
        throw std::invalid_argument("division: requires deg a >= deg b >= 0");
    canonical(a, F, "division dividend");
    canonical(b, F, "division divisor");
    if (block_param < 1) throw std::invalid_argument("division: block parameter must be >= 1");
    if (variant == Variant::naive && 2 * block_param > mp.Z)
        throw std::invalid_argument("division: naive variant requires 2*ell <= Z");
    if (variant == Variant::optimized && 7 * block_param > mp.Z)
        throw std::invalid_argument("division: optimized variant requires 7*s <= Z");
    const std::int64_t s = variant == Variant::naive ? 1 : block_param;  // one head per step
    Clock clk;
    DivisionResult res;
    std::tie(res.q, res.r) = gpu_divmod(a, b, F, s);
    res.sim = clk.report(s);
    if (testhooks::corrupt_division_output && !res.q.is_zero())
        res.q.c[0] = F.add(res.q.c[0], 1);
    return res;
}

GcdResult run_gcd(Variant variant, const MachineParams& mp, const Field& F, const Poly& a_in,
                  const Poly& b_in, std::int64_t block_param) {
    const Poly a = trimmed(a_in), b = trimmed(b_in);
    if (b.is_zero()) throw std::invalid_argument("gcd: second operand must be nonzero");
    if (a.is_zero() || a.degree() < b.degree())
        throw std::invalid_argument("gcd: requires deg a >= deg b >= 0");
    canonical(a, F, "gcd first operand");
    canonical(b, F, "gcd second operand");
    if (variant == Variant::naive) {
        if (block_param < 1) throw std::invalid_argument("gcd: ell must be >= 1");
        if (2 * block_param > mp.Z)
            throw std::invalid_argument("gcd: naive variant requires 2*ell <= Z");
    } else {
        if (block_param < 2) throw std::invalid_argument("gcd: optimized variant requires s >= 2");
        if (6 * block_param > mp.Z)
            throw std::invalid_argument("gcd: optimized variant requires 6*s <= Z");
    }
    const std::int64_t s = variant == Variant::naive ? 1 : block_param;
    Clock clk;
    GcdResult res;
    res.g = gpu_gcd(a, b, F, s);
    res.sim = clk.report(s);
    return res;
}

}  // namespace mmm
