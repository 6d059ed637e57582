// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" face over the UNMODIFIED reference oracle, compiled from the
// sources where they lie (/root/reference/proj/src/{field,poly,oracle}.cpp)
// by oracle/Makefile into oracle/_ref/libref_oracle.so.  Used to pin the C
// restatement (oracle.c) and as the reference CPU arm of bench.py.  Same
// argument conventions as oracle.h (int64 residues, trimmed lengths).
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <vector>

#include "mmm/field.hpp"
#include "mmm/oracle.hpp"
#include "mmm/poly.hpp"

namespace {

mmm::Poly mk(const std::int64_t* c, std::int64_t n) {
    return mmm::Poly(std::vector<std::int64_t>(c, c + n));
}

std::int64_t put(const mmm::Poly& p, std::int64_t* out) {
    if (!p.c.empty()) std::memcpy(out, p.c.data(), p.c.size() * sizeof(std::int64_t));
    return static_cast<std::int64_t>(p.c.size());
}

template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::domain_error&) {
        return 2;
    }
}

}  // namespace

extern "C" {

int ref_field_check(std::int64_t p) {
    return guarded([&] { mmm::Field F(p); });
}

std::int64_t ref_inv(std::int64_t a, std::int64_t p) {
    std::int64_t r = -1;
    guarded([&] { r = mmm::Field(p).inv(a); });
    return r;
}

void* ref_rng_new(std::uint64_t seed) { return new std::mt19937_64(seed); }
void ref_rng_free(void* g) { delete static_cast<std::mt19937_64*>(g); }
std::uint64_t ref_rng_next(void* g) { return (*static_cast<std::mt19937_64*>(g))(); }

int ref_random_poly(void* g, std::int64_t terms, std::int64_t p, std::int64_t* out) {
    return guarded([&] {
        mmm::Field F(p);
        put(mmm::random_poly(*static_cast<std::mt19937_64*>(g), terms, F), out);
    });
}

std::int64_t ref_mul(const std::int64_t* a, std::int64_t na, const std::int64_t* b,
                     std::int64_t nb, std::int64_t p, std::int64_t* out) {
    return put(mmm::oracle_mul(mk(a, na), mk(b, nb), mmm::Field(p)), out);
}

std::int64_t ref_mul_alt(const std::int64_t* a, std::int64_t na, const std::int64_t* b,
                         std::int64_t nb, std::int64_t p, std::int64_t* out) {
    return put(mmm::oracle_mul_alt(mk(a, na), mk(b, nb), mmm::Field(p)), out);
}

int ref_divmod(const std::int64_t* a, std::int64_t na, const std::int64_t* b, std::int64_t nb,
               std::int64_t p, std::int64_t* q, std::int64_t* nq, std::int64_t* r,
               std::int64_t* nr) {
    return guarded([&] {
        auto qr = mmm::oracle_divmod(mk(a, na), mk(b, nb), mmm::Field(p));
        *nq = put(qr.first, q);
        *nr = put(qr.second, r);
    });
}

int ref_gcd(const std::int64_t* a, std::int64_t na, const std::int64_t* b, std::int64_t nb,
            std::int64_t p, std::int64_t* g, std::int64_t* ng) {
    return guarded([&] { *ng = put(mmm::oracle_gcd(mk(a, na), mk(b, nb), mmm::Field(p)), g); });
}

}  // extern "C"
