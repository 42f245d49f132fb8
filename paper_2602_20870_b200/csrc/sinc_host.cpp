// sinc_host.cpp -- host-side series coefficients and content fingerprint for the product
// library. Restates proj/include/fgfrft/sinc.hpp:15-63 and rng.hpp:59-67 term for term and is
// compiled with -ffp-contract=off against the same libm, so coefficients are bit-identical
// to the reference's (pinned in tests/test_capi.py against oracle/_ref and the golden vectors).
// Coefficients are evaluated here, never on the device: device sin/cos differ in the last ulp,
// which would break the exact-Kronecker integer orders and the c_n(-a) = c_{-n}(a) parity.
#include <cmath>
#include <cstddef>
#include <cstdint>

namespace fgb {

double host_sinc(double x) {
    if (x == std::nearbyint(x)) return x == 0.0 ? 1.0 : 0.0;
    if (std::fabs(x) < 1e-6) {
        const double px = M_PI * x;
        return 1.0 - px * px / 6.0;
    }
    return std::sin(M_PI * x) / (M_PI * x);
}

double host_sinc_deriv(double x) {
    if (x == std::nearbyint(x)) {
        if (x == 0.0) return 0.0;
        const long long k = static_cast<long long>(x);
        return (k % 2 == 0 ? 1.0 : -1.0) / x;
    }
    if (std::fabs(x) < 1e-6) {
        const double pi2 = M_PI * M_PI;
        return -pi2 * x / 3.0 + pi2 * pi2 * x * x * x / 30.0;
    }
    const double px = M_PI * x;
    return std::cos(px) / x - std::sin(px) / (M_PI * x * x);
}

// Both tables at once: the generic branch of sinc and sinc' shares one sin(pi x) and one
// cos(pi x) evaluation per term (the same libm calls on the same argument as host_sinc /
// host_sinc_deriv, so the values are bit-identical to evaluating them separately).
void host_sinc_coeffs(double alpha, int l, double* c, double* dc) {
    for (int n = -l; n <= l; ++n) {
        const double x = alpha - static_cast<double>(n);
        if (x == std::nearbyint(x) || std::fabs(x) < 1e-6) {
            if (c) c[n + l] = host_sinc(x);
            if (dc) dc[n + l] = host_sinc_deriv(x);
            continue;
        }
        const double px = M_PI * x;
        const double sn = std::sin(px);
        if (c) c[n + l] = sn / (M_PI * x);
        if (dc) dc[n + l] = std::cos(px) / x - sn / (M_PI * x * x);
    }
}

// The same coefficients from ONE sin / cos per order: sin(pi (a - n)) = (-1)^(m - n) sin(pi f) with
// a = m + f, |f| <= 1/2 -- more accurate than the reference's per-term sin(M_PI * x) (whose argument
// carries |x| ulp of rounding) and ~15x cheaper. For the host-side planning tables of the node
// and order-window routes only (interpolation checks, node operators); the tables the synthesis
// kernels consume stay host_sinc_coeffs, bit-identical to sinc.hpp.
void host_sinc_coeffs_fast(double alpha, int l, double* c, double* dc) {
    const double m = std::nearbyint(alpha), f = alpha - m;
    const double s = std::sin(M_PI * f), co = std::cos(M_PI * f);
    const long long mi = static_cast<long long>(m);
    for (int n = -l; n <= l; ++n) {
        const double x = alpha - static_cast<double>(n);
        if (x == std::nearbyint(x) || std::fabs(x) < 1e-6) {
            if (c) c[n + l] = host_sinc(x);
            if (dc) dc[n + l] = host_sinc_deriv(x);
            continue;
        }
        const double sg = ((mi - n) & 1) ? -1.0 : 1.0;
        const double sn = sg * s, cs = sg * co;
        if (c) c[n + l] = sn / (M_PI * x);
        if (dc) dc[n + l] = cs / x - sn / (M_PI * x * x);
    }
}

uint64_t host_fnv1a64(const void* data, size_t nbytes) {
    const auto* p = static_cast<const unsigned char*>(data);
    uint64_t h = 0xcbf29ce484222325ULL;
    for (size_t i = 0; i < nbytes; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

}  // namespace fgb
