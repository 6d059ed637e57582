// mmm_verify.cpp -- GPU counterpart of `mmm verify` (proj/tools/mmm_cli.cpp:456-528):
// random instances drawn in the reference's order, every kernel program run
// through the C++ drop-in on the B200, checked against the C oracle
// restatement.  Flags: --app all|division|multiplication|gcd --trials N
// --seed S --p P --Z Z --max-n N --inject-fault.  Exit 0 all ok, 2 mismatch,
// 1 usage/runtime error (the reference's codes, mmm_cli.cpp:6-7).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <random>
#include <string>

#include "../../include/mmm_b200.hpp"
#include "../../oracle/oracle.h"

using mmm::Field;
using mmm::Poly;
using mmm::Variant;

namespace {

std::int64_t pick(std::mt19937_64& rng, std::int64_t lo, std::int64_t hi) {
    return lo + static_cast<std::int64_t>(rng() % static_cast<std::uint64_t>(hi - lo + 1));
}

Poly o_mul(const Poly& a, const Poly& b, const Field& F) {
    std::vector<int64_t> out(a.c.size() + b.c.size() + 1);
    out.resize(size_t(orc_poly_mul(a.c.data(), int64_t(a.c.size()), b.c.data(),
                                   int64_t(b.c.size()), F.p(), out.data())));
    return Poly(out);
}
Poly o_add(const Poly& a, const Poly& b, const Field& F) {
    std::vector<int64_t> out(std::max(a.c.size(), b.c.size()) + 1);
    out.resize(size_t(orc_poly_add(a.c.data(), int64_t(a.c.size()), b.c.data(),
                                   int64_t(b.c.size()), F.p(), out.data())));
    return Poly(out);
}
std::pair<Poly, Poly> o_divmod(const Poly& a, const Poly& b, const Field& F) {
    std::vector<int64_t> q(a.c.size() + 1), r(a.c.size() + 1);
    int64_t nq = 0, nr = 0;
    orc_divmod(a.c.data(), int64_t(a.c.size()), b.c.data(), int64_t(b.c.size()), F.p(), q.data(),
               &nq, r.data(), &nr);
    q.resize(size_t(nq));
    r.resize(size_t(nr));
    return {Poly(q), Poly(r)};
}
Poly o_gcd(const Poly& a, const Poly& b, const Field& F) {
    std::vector<int64_t> g(std::max(a.c.size(), b.c.size()) + 1);
    int64_t ng = 0;
    orc_gcd(a.c.data(), int64_t(a.c.size()), b.c.data(), int64_t(b.c.size()), F.p(), g.data(), &ng);
    g.resize(size_t(ng));
    return Poly(g);
}

}  // namespace

int main(int argc, char** argv) {
    std::string app = "all";
    std::int64_t trials = 200, p = 101, Z = 1024, max_n = 64;
    std::uint64_t seed = 42;
    bool inject = false;
    for (int i = 1; i < argc; ++i) {
        const std::string k = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) {
                std::cerr << "verify: " << k << " needs a value\n";
                std::exit(1);
            }
            return argv[++i];
        };
        if (k == "--app") app = val();
        else if (k == "--trials") trials = std::stoll(val());
        else if (k == "--seed") seed = std::stoull(val());
        else if (k == "--p") p = std::stoll(val());
        else if (k == "--Z") Z = std::stoll(val());
        else if (k == "--max-n") max_n = std::stoll(val());
        else if (k == "--inject-fault") inject = true;
        else {
            std::cerr << "verify: unknown option " << k << "\n";
            return 1;
        }
    }
    if (trials < 1 || max_n < 1 || Z < 15) {
        std::cerr << "verify: requires --trials >= 1, --max-n >= 1, --Z >= 15\n";
        return 1;
    }
    try {
        const bool run_div = app == "all" || app == "division";
        const bool run_mul = app == "all" || app == "multiplication";
        const bool run_gcd = app == "all" || app == "gcd";
        const Field F(p);
        mmm::MachineParams mp;
        mp.Z = Z;
        std::mt19937_64 rng(seed);
        mmm::testhooks::corrupt_division_output = inject;
        std::int64_t div_ok = 0, mul_ok = 0, gcd_ok = 0, fails = 0;
        for (std::int64_t t = 0; t < trials; ++t) {
            const std::int64_t m = pick(rng, 1, max_n);
            const std::int64_t n = pick(rng, m, max_n);
            const std::int64_t nm = pick(rng, 1, max_n);
            const std::int64_t l = pick(rng, 1, std::min<std::int64_t>(8, Z / 2));
            const std::int64_t s_div = pick(rng, 1, std::min<std::int64_t>(8, Z / 7));
            const std::int64_t s_gcd = pick(rng, 2, std::min<std::int64_t>(8, Z / 6));
            const Poly a = mmm::random_poly(rng, n, F);
            const Poly b = mmm::random_poly(rng, m, F);
            const Poly am = mmm::random_poly(rng, nm, F);
            if (run_div) {
                const auto nv = mmm::run_division(Variant::naive, mp, F, a, b, l);
                const auto op = mmm::run_division(Variant::optimized, mp, F, a, b, s_div);
                const auto want = o_divmod(a, b, F);
                const bool ok = nv.q == op.q && nv.r == op.r && nv.q == want.first &&
                                nv.r == want.second && o_add(o_mul(nv.q, b, F), nv.r, F) == a &&
                                nv.r.degree() < b.degree();
                if (ok) ++div_ok;
                else {
                    ++fails;
                    std::cerr << "verify: division mismatch at trial " << t << " (n=" << n
                              << ", m=" << m << ")\n";
                }
            }
            if (run_mul) {
                bool ok = true;
                const Poly want = o_mul(am, b, F);
                for (std::int64_t s : {1, 2, 4}) {
                    const std::int64_t lw = std::min<std::int64_t>(l, (Z - 2 * s + 1) / (2 * s));
                    ok = ok && mmm::run_multiplication(mp, F, am, b, s,
                                                       std::max<std::int64_t>(1, lw)).f == want;
                }
                if (ok) ++mul_ok;
                else {
                    ++fails;
                    std::cerr << "verify: multiplication mismatch at trial " << t << "\n";
                }
            }
            if (run_gcd) {
                const Poly want = o_gcd(a, b, F);
                const bool ok = mmm::run_gcd(Variant::naive, mp, F, a, b, l).g == want &&
                                mmm::run_gcd(Variant::optimized, mp, F, a, b, s_gcd).g == want;
                if (ok) ++gcd_ok;
                else {
                    ++fails;
                    std::cerr << "verify: gcd mismatch at trial " << t << "\n";
                }
            }
        }
        if (run_div) std::cout << "division: " << div_ok << "/" << trials << " ok\n";
        if (run_mul) std::cout << "multiplication: " << mul_ok << "/" << trials << " ok\n";
        if (run_gcd) std::cout << "gcd: " << gcd_ok << "/" << trials << " ok\n";
        return fails == 0 ? 0 : 2;
    } catch (const std::exception& e) {
        std::cerr << "verify: " << e.what() << "\n";
        return 1;
    }
}
