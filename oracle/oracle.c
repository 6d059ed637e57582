/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain-C restatement of the reference's serial path.  Each function cites
 * the reference lines it restates (paths relative to /root/reference/proj).
 * Nothing here is optimised: it is the checker and the CPU baseline.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- field -- */

/* field.cpp:10-16 (is_prime) and field.cpp:20-25 (constructor checks). */
int orc_field_check(int64_t p) {
    if (p < 2 || p >= ((int64_t)1 << 31)) return ORC_INVALID_ARGUMENT;
    if (p % 2 == 0) return p == 2 ? ORC_OK : ORC_INVALID_ARGUMENT;
    for (int64_t d = 3; d * d <= p; d += 2)
        if (p % d == 0) return ORC_INVALID_ARGUMENT;
    return ORC_OK;
}

/* field.hpp:15-22: conditional +-p on canonical inputs. */
int64_t orc_add(int64_t a, int64_t b, int64_t p) {
    int64_t s = a + b;
    return s >= p ? s - p : s;
}
int64_t orc_sub(int64_t a, int64_t b, int64_t p) {
    int64_t s = a - b;
    return s < 0 ? s + p : s;
}
/* field.hpp:23: (a*b) % p on int64. */
int64_t orc_mulmod(int64_t a, int64_t b, int64_t p) { return (a * b) % p; }
/* field.hpp:32-35. */
int64_t orc_reduce(int64_t x, int64_t p) {
    int64_t r = x % p;
    return r < 0 ? r + p : r;
}
/* field.cpp:27-42: extended Euclid on (a, p). */
int64_t orc_inv(int64_t a, int64_t p) {
    if (a == 0) return -1;
    int64_t old_r = a, r = p, old_t = 1, t = 0;
    while (r != 0) {
        int64_t q = old_r / r, tmp = old_r - q * r;
        old_r = r;
        r = tmp;
        tmp = old_t - q * t;
        old_t = t;
        t = tmp;
    }
    return orc_reduce(old_t, p);
}

/* ------------------------------------------------------- mt19937_64 ------ */
/* The published MT19937-64 recurrence (Matsumoto & Nishimura), parameters of
 * std::mt19937_64 (C++ [rand.predef]). */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void orc_mt_seed(orc_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = MT_N;
}

static void mt_twist(orc_mt64* g) {
    for (int i = 0; i < MT_N; ++i) {
        uint64_t x = (g->mt[i] & MT_UPPER) | (g->mt[(i + 1) % MT_N] & MT_LOWER);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= MT_A;
        g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ xa;
    }
    g->idx = 0;
}

uint64_t orc_mt_next(orc_mt64* g) {
    if (g->idx >= MT_N) mt_twist(g);
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* uniform_int_distribution<int64_t>{lo, hi} as libstdc++ (GCC 13) draws it
 * from a full-range 64-bit engine: Lemire's nearly-divisionless downscale
 * ("Fast Random Integer Generation in an Interval", 2019) over range+1. */
int64_t orc_uniform(orc_mt64* g, int64_t lo, int64_t hi) {
    uint64_t range = (uint64_t)hi - (uint64_t)lo;
    if (range == UINT64_MAX) return (int64_t)orc_mt_next(g);
    uint64_t erange = range + 1;
    unsigned __int128 prod = (unsigned __int128)orc_mt_next(g) * erange;
    uint64_t low = (uint64_t)prod;
    if (low < erange) {
        uint64_t threshold = (0 - erange) % erange;
        while (low < threshold) {
            prod = (unsigned __int128)orc_mt_next(g) * erange;
            low = (uint64_t)prod;
        }
    }
    return (int64_t)((uint64_t)(prod >> 64) + (uint64_t)lo);
}

/* poly.cpp:20-29. */
int orc_random_poly(orc_mt64* g, int64_t terms, int64_t p, int64_t* out) {
    if (terms < 1) return ORC_INVALID_ARGUMENT;
    for (int64_t i = 0; i + 1 < terms; ++i) out[i] = orc_uniform(g, 0, p - 1);
    out[terms - 1] = orc_uniform(g, 1, p - 1);
    return ORC_OK;
}

/* ------------------------------------------------------------- poly ------ */

/* poly.cpp:7-10. */
int64_t orc_trim(const int64_t* c, int64_t len) {
    while (len > 0 && c[len - 1] == 0) --len;
    return len;
}

/* poly.cpp:12-18. */
int64_t orc_monic(const int64_t* a, int64_t na, int64_t p, int64_t* out) {
    na = orc_trim(a, na);
    if (na == 0) return 0;
    int64_t s = orc_inv(a[na - 1], p);
    for (int64_t i = 0; i < na; ++i) out[i] = orc_mulmod(a[i], s, p);
    return na;
}

/* oracle.cpp:8-15: iterate input index pairs. */
int64_t orc_poly_mul(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p,
                     int64_t* out) {
    if (na == 0 || nb == 0) return 0;
    int64_t nf = na + nb - 1;
    memset(out, 0, (size_t)nf * sizeof(int64_t));
    for (int64_t i = 0; i < na; ++i)
        for (int64_t j = 0; j < nb; ++j)
            out[i + j] = orc_add(out[i + j], orc_mulmod(a[i], b[j], p), p);
    return orc_trim(out, nf);
}

/* oracle.cpp:17-29: output-stationary. */
int64_t orc_poly_mul_alt(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p,
                         int64_t* out) {
    if (na == 0 || nb == 0) return 0;
    int64_t nf = na + nb - 1;
    for (int64_t k = 0; k < nf; ++k) {
        int64_t acc = 0;
        int64_t lo = k >= nb - 1 ? k - (nb - 1) : 0;
        int64_t hi = k < na - 1 ? k : na - 1;
        for (int64_t i = lo; i <= hi; ++i) acc = orc_add(acc, orc_mulmod(a[i], b[k - i], p), p);
        out[k] = acc;
    }
    return orc_trim(out, nf);
}

/* oracle_mul_alt restricted to output words [k0, k1) (untrimmed): lets the
 * test harness split one large golden product across host threads. */
void orc_poly_mul_alt_range(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p,
                            int64_t k0, int64_t k1, int64_t* out) {
    for (int64_t k = k0; k < k1; ++k) {
        int64_t acc = 0;
        int64_t lo = k >= nb - 1 ? k - (nb - 1) : 0;
        int64_t hi = k < na - 1 ? k : na - 1;
        for (int64_t i = lo; i <= hi; ++i) acc = orc_add(acc, orc_mulmod(a[i], b[k - i], p), p);
        out[k - k0] = acc;
    }
}

/* oracle.cpp:31-49. */
static int64_t addsub(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p,
                      int64_t* out, int neg) {
    int64_t n = na > nb ? na : nb;
    for (int64_t i = 0; i < n; ++i) {
        int64_t va = i < na ? a[i] : 0, vb = i < nb ? b[i] : 0;
        out[i] = neg ? orc_sub(va, vb, p) : orc_add(va, vb, p);
    }
    return orc_trim(out, n);
}
int64_t orc_poly_add(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p,
                     int64_t* out) {
    return addsub(a, na, b, nb, p, out, 0);
}
int64_t orc_poly_sub(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p,
                     int64_t* out) {
    return addsub(a, na, b, nb, p, out, 1);
}

/* In-place remainder of r (length nr, trimmed) by b (trimmed, nonzero):
 * the j-loop of oracle.cpp:63-64, skipping zero heads (oracle.cpp:60).
 * Quotient words go to q when q != NULL.  Counts eliminations/updates. */
static int64_t rem_inplace(int64_t* r, int64_t nr, const int64_t* b, int64_t nb, int64_t p,
                           int64_t* q, int64_t* steps, int64_t* updates) {
    int64_t db = nb - 1;
    int64_t lead_inv = orc_inv(b[db], p);
    for (int64_t i = nr - 1; i >= db; --i) {
        int64_t cur = r[i];
        if (cur == 0) continue;
        int64_t coef = orc_mulmod(cur, lead_inv, p);
        if (q) q[i - db] = coef;
        for (int64_t j = 0; j <= db; ++j)
            r[i - db + j] = orc_sub(r[i - db + j], orc_mulmod(coef, b[j], p), p);
        if (steps) ++*steps;
        if (updates) *updates += db + 1;
    }
    return orc_trim(r, nr < db ? nr : db);
}

/* oracle.cpp:51-67. */
int orc_divmod(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p, int64_t* q,
               int64_t* nq, int64_t* r, int64_t* nr) {
    /* b is used as given (not trimmed), exactly like oracle.cpp:52-55; a
     * non-canonical b with a zero lead fails in Field::inv (field.cpp:28). */
    if (nb == 0) return ORC_DOMAIN_ERROR;
    na = orc_trim(a, na);
    memcpy(r, a, (size_t)na * sizeof(int64_t));
    if (na < nb) {
        *nq = 0;
        *nr = na;
        return ORC_OK;
    }
    if (b[nb - 1] == 0) return ORC_DOMAIN_ERROR;
    int64_t lq = na - nb + 1;
    memset(q, 0, (size_t)lq * sizeof(int64_t));
    *nr = rem_inplace(r, na, b, nb, p, q, NULL, NULL);
    *nq = orc_trim(q, lq);
    return ORC_OK;
}

static int euclid(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p,
                  int64_t* g, int64_t* ng, int64_t* steps, int64_t* updates) {
    na = orc_trim(a, na);
    nb = orc_trim(b, nb);
    if (na == 0 && nb == 0) return ORC_DOMAIN_ERROR;
    int64_t cap = (na > nb ? na : nb) + 1;
    int64_t* x = (int64_t*)malloc((size_t)cap * sizeof(int64_t));
    int64_t* y = (int64_t*)malloc((size_t)cap * sizeof(int64_t));
    memcpy(x, a, (size_t)na * sizeof(int64_t));
    memcpy(y, b, (size_t)nb * sizeof(int64_t));
    int64_t nx = na, ny = nb;
    /* oracle.cpp:72-76: x, y <- y, x mod y until y vanishes. */
    while (ny != 0) {
        int64_t nr = nx < ny ? nx : rem_inplace(x, nx, y, ny, p, NULL, steps, updates);
        int64_t* t = x;
        x = y;
        nx = ny;
        y = t;
        ny = nr;
    }
    if (g) *ng = orc_monic(x, nx, p, g); /* oracle.cpp:77 */
    free(x);
    free(y);
    return ORC_OK;
}

/* oracle.cpp:69-78. */
int orc_gcd(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p, int64_t* g,
            int64_t* ng) {
    return euclid(a, na, b, nb, p, g, ng, NULL, NULL);
}

int orc_gcd_count(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p,
                  int64_t* steps, int64_t* updates) {
    *steps = 0;
    *updates = 0;
    return euclid(a, na, b, nb, p, NULL, NULL, steps, updates);
}
