// ref_shim.cpp -- TEST INFRASTRUCTURE. Compiles the reference's own std-only headers
// (sinc.hpp, rng.hpp, errors.hpp) where they lie under /root/reference and exposes them
// through a C ABI so the oracle restatement and the input generators can be pinned
// bit-for-bit against the reference. transform.hpp / gft.hpp / spectral.hpp need Eigen3,
// which is absent (no network), so they cannot be built here.
// Built by oracle/Makefile into oracle/_ref/libfgfrft_ref_shim.so; never shipped in the product.
#include <cstdint>
#include <cstring>
#include "fgfrft/sinc.hpp"
#include "fgfrft/rng.hpp"

extern "C" {

int ref_sinc_coeffs(double alpha, int l, double* c, double* dc) {
    try {
        const fgfrft::SincCoeffs s = fgfrft::sinc_coeffs(alpha, l);
        std::memcpy(c, s.c.data(), s.c.size() * sizeof(double));
        std::memcpy(dc, s.dc.data(), s.dc.size() * sizeof(double));
        return 0;
    } catch (const fgfrft::parameter_error&) {
        return -1;
    }
}

double ref_sinc(double x) { return fgfrft::sinc(x); }
double ref_sinc_deriv(double x) { return fgfrft::sinc_deriv(x); }

uint64_t ref_fnv1a64(const void* data, size_t nbytes) { return fgfrft::fnv1a64(data, nbytes); }

uint64_t ref_rng_derive(uint64_t seed, uint64_t index) { return fgfrft::Rng::derive(seed, index); }

// kinds: 0 = uniform(), 1 = gaussian(); one kind per output element, same Rng object.
void ref_rng_stream(uint64_t seed, const int* kinds, int64_t n, double* out) {
    fgfrft::Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = kinds[i] == 0 ? rng.uniform() : rng.gaussian();
}

}  // extern "C"
