// test_dropin.cpp -- the reference's unit-test cases, restated against the
// C++ drop-in (include/mmm_b200.hpp -> libmmm_b200.so -> sm_100a kernels),
// with the C oracle restatement (oracle/oracle.h) as the checker.
// Cases follow proj/tests/test_{field,poly_oracle,division,multiplication,gcd}.cpp.
// Exit status 0 iff every CHECK held.
#include <cstdio>
#include <random>
#include <stdexcept>

#include "../../include/mmm_b200.hpp"
#include "../../oracle/oracle.h"

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                                  \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(c)) {                                                               \
            ++g_fail;                                                             \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #c); \
        }                                                                         \
    } while (0)
#define CHECK_THROWS_AS(expr, E)            \
    do {                                    \
        bool thrown = false;                \
        try {                               \
            (void)(expr);                   \
        } catch (const E&) {                \
            thrown = true;                  \
        } catch (...) {                     \
        }                                   \
        CHECK(thrown && #E);                \
    } while (0)

using mmm::Field;
using mmm::MachineParams;
using mmm::Poly;
using mmm::Rat;
using mmm::Variant;

static MachineParams params(Rat U = Rat(4), std::int64_t Z = 1024) {
    MachineParams mp;
    mp.U = U;
    mp.Z = Z;
    return mp;
}

// checker: the C restatement of the reference oracle
static Poly ref_mul(const Poly& a, const Poly& b, const Field& F) {
    std::vector<int64_t> out(a.c.size() + b.c.size() + 1);
    int64_t n = orc_poly_mul(a.c.data(), int64_t(a.c.size()), b.c.data(), int64_t(b.c.size()),
                             F.p(), out.data());
    out.resize(size_t(n));
    return Poly(out);
}
static std::pair<Poly, Poly> ref_divmod(const Poly& a, const Poly& b, const Field& F) {
    std::vector<int64_t> q(a.c.size() + 1), r(a.c.size() + 1);
    int64_t nq = 0, nr = 0;
    orc_divmod(a.c.data(), int64_t(a.c.size()), b.c.data(), int64_t(b.c.size()), F.p(), q.data(),
               &nq, r.data(), &nr);
    q.resize(size_t(nq));
    r.resize(size_t(nr));
    return {Poly(q), Poly(r)};
}
static Poly ref_gcd(const Poly& a, const Poly& b, const Field& F) {
    std::vector<int64_t> g(std::max(a.c.size(), b.c.size()) + 1);
    int64_t ng = 0;
    orc_gcd(a.c.data(), int64_t(a.c.size()), b.c.data(), int64_t(b.c.size()), F.p(), g.data(), &ng);
    g.resize(size_t(ng));
    return Poly(g);
}

static void field_cases() {  // test_field.cpp
    CHECK(Field(7).p() == 7 && Field(2).p() == 2 && Field(469762049).p() == 469762049);
    CHECK_THROWS_AS(Field(6), std::invalid_argument);
    CHECK_THROWS_AS(Field(1), std::invalid_argument);
    CHECK_THROWS_AS(Field(std::int64_t{1} << 31), std::invalid_argument);
    Field F(7);
    CHECK(F.inv(3) == 5 && F.divide(6, 2) == 3 && F.reduce(-1) == 6);
    CHECK_THROWS_AS(Field(101).inv(0), std::domain_error);
    Field G(2147483647);
    CHECK(G.mul(2147483646, 2147483646) == 1 && G.inv(2147483646) == 2147483646);
}

static void poly_cases() {  // test_poly_oracle.cpp
    Field F(7);
    CHECK(mmm::to_string(Poly{5, 0, 3}) == "3*X^2 + 5" && mmm::to_string(Poly{}) == "0");
    CHECK(mmm::trimmed(Poly{1, 2, 0, 0}) == (Poly{1, 2}));
    CHECK(mmm::monic(Poly{2, 4}, F) == (Poly{4, 1}));
    auto qr = mmm::oracle_divmod(Poly{1, 2, 0, 1}, Poly{1, 1}, F);
    CHECK(qr.first == (Poly{3, 6, 1}) && qr.second == (Poly{5}));
    CHECK_THROWS_AS(mmm::oracle_divmod(Poly{3, 0, 2, 5}, Poly{}, F), std::domain_error);
    CHECK(mmm::oracle_mul(Poly{1, 1}, Poly{1, 1}, F) == (Poly{1, 2, 1}));
    CHECK(mmm::oracle_mul(Poly{2, 5, 1}, Poly{}, F) == Poly{});
    CHECK(mmm::oracle_gcd(Poly{2, 3, 1}, Poly{3, 4, 1}, F) == (Poly{1, 1}));
    CHECK_THROWS_AS(mmm::oracle_gcd(Poly{}, Poly{}, F), std::domain_error);
    std::mt19937_64 rng(2026);
    Field F7(7), F101(101), Fp(469762049);
    for (int t = 0; t < 200; ++t) {
        const Field& G = t % 3 == 0 ? F7 : (t % 3 == 1 ? F101 : Fp);
        std::int64_t n = 1 + std::int64_t(rng() % 20), m = 1 + std::int64_t(rng() % 20);
        Poly a = mmm::random_poly(rng, n, G), b = mmm::random_poly(rng, m, G);
        Poly f = mmm::oracle_mul(a, b, G);
        CHECK(f == ref_mul(a, b, G));
        CHECK(mmm::oracle_mul_alt(a, b, G) == f);  // NTT path where p allows
    }
}

static void division_cases() {  // test_division.cpp
    Field F(7);
    Poly a{1, 2, 0, 1}, b{1, 1};
    auto naive = mmm::run_division(Variant::naive, params(), F, a, b, 4);
    CHECK(naive.q == (Poly{3, 6, 1}) && naive.r == (Poly{5}));
    for (std::int64_t s : {1, 2}) {
        auto opt = mmm::run_division(Variant::optimized, params(), F, a, b, s);
        CHECK(opt.q == naive.q && opt.r == naive.r);
    }
    Field F101(101);
    Poly c{3, 0, 7, 1};
    CHECK_THROWS_AS(mmm::run_division(Variant::naive, params(), F101, c, Poly{}, 4),
                    std::invalid_argument);
    CHECK_THROWS_AS(mmm::run_division(Variant::naive, params(), F101, Poly{1, 2}, c, 4),
                    std::invalid_argument);
    CHECK_THROWS_AS(mmm::run_division(Variant::naive, params(), F101, c, c, 0),
                    std::invalid_argument);
    CHECK_THROWS_AS(mmm::run_division(Variant::naive, params(Rat(4), 6), F101, c, c, 4),
                    std::invalid_argument);
    CHECK_THROWS_AS(mmm::run_division(Variant::optimized, params(Rat(4), 13), F101, c, c, 2),
                    std::invalid_argument);
    Poly x5{1, 0, 0, 0, 0, 1}, x2{1, 0, 1};
    auto oqr = ref_divmod(x5, x2, F);
    for (std::int64_t s : {1, 2, 3}) {
        auto opt = mmm::run_division(Variant::optimized, params(), F, x5, x2, s);
        CHECK(opt.q == oqr.first && opt.r == oqr.second);
    }
    std::mt19937_64 rng(424242);
    for (std::int64_t p : {7, 101}) {
        Field G(p);
        for (int t = 0; t < 20; ++t) {
            std::int64_t m = 1 + std::int64_t(rng() % 20);
            std::int64_t n = m + std::int64_t(rng() % 30);
            Poly A = mmm::random_poly(rng, n, G), B = mmm::random_poly(rng, m, G);
            auto want = ref_divmod(A, B, G);
            auto nv = mmm::run_division(Variant::naive, params(), G, A, B, 4);
            CHECK(nv.q == want.first && nv.r == want.second);
            for (std::int64_t s : {1, 2, 3, 4, 8}) {
                auto opt = mmm::run_division(Variant::optimized, params(), G, A, B, s);
                CHECK(opt.q == want.first && opt.r == want.second);
            }
            CHECK(mmm::oracle_add(mmm::oracle_mul(nv.q, B, G), nv.r, G) == A);
        }
    }
}

static void multiplication_cases() {  // test_multiplication.cpp
    Field F(7);
    CHECK(mmm::run_multiplication(params(), F, Poly{1, 1}, Poly{1, 1}, 1, 4).f == (Poly{1, 2, 1}));
    CHECK(mmm::run_multiplication(params(), F, Poly{3}, Poly{2, 5, 1}, 1, 4).f == (Poly{6, 1, 3}));
    Poly a{1, 1};
    CHECK_THROWS_AS(mmm::run_multiplication(params(), F, Poly{}, a, 1, 4), std::invalid_argument);
    CHECK_THROWS_AS(mmm::run_multiplication(params(), F, a, a, 0, 4), std::invalid_argument);
    CHECK_THROWS_AS(mmm::run_multiplication(params(), F, a, a, 1, 0), std::invalid_argument);
    CHECK_THROWS_AS(mmm::run_multiplication(params(Rat(4), 18), F, a, a, 2, 4),
                    std::invalid_argument);
    CHECK(mmm::run_multiplication(params(Rat(4), 19), F, a, a, 2, 4).f == (Poly{1, 2, 1}));
    std::mt19937_64 rng(1337);
    for (std::int64_t p : {7, 101}) {
        Field G(p);
        for (int t = 0; t < 15; ++t) {
            std::int64_t n = 1 + std::int64_t(rng() % 40), m = 1 + std::int64_t(rng() % 40);
            Poly A = mmm::random_poly(rng, n, G), B = mmm::random_poly(rng, m, G);
            Poly want = ref_mul(A, B, G);
            for (std::int64_t s : {1, 2, 3, 4, 8})
                for (std::int64_t l : {1, 4, 16}) {
                    auto res = mmm::run_multiplication(params(), G, A, B, s, l);
                    CHECK(res.f == want);
                    CHECK(!res.sim.kernels.empty());
                    CHECK(res.sim.metrics.structure.L == int64_t(res.sim.kernels.size()));
                    CHECK(res.sim.metrics.structure.N >= res.sim.metrics.structure.K);
                    CHECK(res.sim.metrics.structure.K >= 1);
                    CHECK(res.sim.kernels[0].name.rfind("mul_kernel", 0) == 0);
                }
        }
    }
}

static void gcd_cases() {  // test_gcd.cpp
    Field F(7);
    CHECK(mmm::run_gcd(Variant::naive, params(), F, Poly{2, 3, 1}, Poly{3, 4, 1}, 4).g ==
          (Poly{1, 1}));
    CHECK(mmm::run_gcd(Variant::optimized, params(), F, Poly{2, 3, 1}, Poly{3, 4, 1}, 2).g ==
          (Poly{1, 1}));
    Poly b{2, 4, 6}, q{1, 0, 5, 1};
    Poly a = ref_mul(b, q, F);
    CHECK(mmm::run_gcd(Variant::naive, params(), F, a, b, 4).g == mmm::monic(b, F));
    CHECK(mmm::run_gcd(Variant::optimized, params(), F, a, b, 2).g == mmm::monic(b, F));
    CHECK(mmm::run_gcd(Variant::naive, params(), F, a, a, 4).g == mmm::monic(a, F));
    CHECK(mmm::run_gcd(Variant::naive, params(), F, ref_mul(Poly{1, 1}, Poly{1, 1}, F),
                       Poly{2, 1}, 4).g == (Poly{1}));
    Field F101(101);
    for (Variant v : {Variant::naive, Variant::optimized})
        CHECK(mmm::run_gcd(v, params(), F101, Poly{42}, Poly{9}, v == Variant::naive ? 4 : 2).g ==
              (Poly{1}));
    Poly x{1, 1, 1}, y{1, 1};
    CHECK_THROWS_AS(mmm::run_gcd(Variant::naive, params(), F, x, Poly{}, 4), std::invalid_argument);
    CHECK_THROWS_AS(mmm::run_gcd(Variant::naive, params(), F, y, x, 4), std::invalid_argument);
    CHECK_THROWS_AS(mmm::run_gcd(Variant::optimized, params(), F, x, y, 1), std::invalid_argument);
    CHECK_THROWS_AS(mmm::run_gcd(Variant::optimized, params(Rat(4), 11), F, x, y, 2),
                    std::invalid_argument);
    std::mt19937_64 rng(4242);
    for (std::int64_t p : {7, 101}) {
        Field G(p);
        for (int t = 0; t < 12; ++t) {
            std::int64_t ta = 1 + std::int64_t(rng() % 24), tb = 1 + std::int64_t(rng() % 24);
            if (ta < tb) std::swap(ta, tb);
            Poly A = mmm::random_poly(rng, ta, G), B = mmm::random_poly(rng, tb, G);
            Poly want = ref_gcd(A, B, G);
            CHECK(mmm::run_gcd(Variant::naive, params(), G, A, B, 4).g == want);
            for (std::int64_t s : {2, 4, 8})
                CHECK(mmm::run_gcd(Variant::optimized, params(), G, A, B, s).g == want);
        }
    }
}

int main() {
    try {
        field_cases();
        poly_cases();
        division_cases();
        multiplication_cases();
        gcd_cases();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "unexpected exception: %s\n", e.what());
        return 1;
    }
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
