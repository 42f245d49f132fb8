/*
 * prep_rng.c -- deterministic input generation (host-side input prep, not the hot path).
 * Restates the reference Rng (proj/include/fgfrft/rng.hpp:12-56): mt19937_64, 53-bit
 * uniform in [0,1), Box-Muller Gaussian with a cached spare, and the splitmix64 derive().
 * Bit-exact against the reference (pinned in tests/test_prep.py via oracle/_ref and the
 * committed golden stream tests/golden/rng_stream.json).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#define MT_N 312
#define MT_M 156

typedef struct {
    uint64_t mt[MT_N];
    int idx;
    double spare;
    int have_spare;
} prep_rng;

static void mt_seed(prep_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
}

static uint64_t mt_next(prep_rng* r) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    if (r->idx >= MT_N) {
        for (int i = 0; i < MT_N; ++i) {
            const uint64_t y = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
            uint64_t v = r->mt[(i + MT_M) % MT_N] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = v;
        }
        r->idx = 0;
    }
    uint64_t x = r->mt[r->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

prep_rng* prep_rng_create(uint64_t seed) {
    prep_rng* r = (prep_rng*)calloc(1, sizeof(prep_rng));
    if (r) mt_seed(r, seed);
    return r;
}

void prep_rng_destroy(prep_rng* r) { free(r); }

uint64_t prep_rng_bits(prep_rng* r) { return mt_next(r); }

double prep_rng_uniform(prep_rng* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }

double prep_rng_gaussian(prep_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1 = prep_rng_uniform(r);
    while (u1 <= 0.0) u1 = prep_rng_uniform(r);
    const double u2 = prep_rng_uniform(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double a = 2.0 * M_PI * u2;
    r->spare = rad * sin(a);
    r->have_spare = 1;
    return rad * cos(a);
}

void prep_rng_fill_uniform(prep_rng* r, int64_t n, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = prep_rng_uniform(r);
}

void prep_rng_fill_gaussian(prep_rng* r, int64_t n, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = prep_rng_gaussian(r);
}

/* Bernoulli(p) draws, one uniform() per output, as the ER generator consumes them. */
void prep_rng_fill_bernoulli(prep_rng* r, int64_t n, double p, unsigned char* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = prep_rng_uniform(r) < p;
}

uint64_t prep_rng_derive(uint64_t seed, uint64_t index) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (index + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
