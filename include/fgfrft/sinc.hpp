#pragma once
// Series weights c_n(alpha) = sinc(alpha - n) and derivatives, n = -L..L (reference:
// proj/include/fgfrft/sinc.hpp:15-63). Evaluated by the library's host code, so the values
// fed to the GPU kernels are exactly the ones returned here (bit-identical to the reference).

#include <cstddef>
#include <vector>

#include "fgfrft/errors.hpp"

#if defined(FGFRFT_HAVE_EIGEN) && __has_include_next(<fgfrft/sinc.hpp>)
// integration builds: the reference's own (std-only, bit-identical) sinc.hpp
#include_next <fgfrft/sinc.hpp>
#else
namespace fgfrft {

struct SincCoeffs {
    double alpha = 0.0;
    int l = 0;
    std::vector<double> c;   // [n + l] = c_n(alpha)
    std::vector<double> dc;  // [n + l] = d c_n / d alpha

    double coeff(int n) const { return c[static_cast<std::size_t>(n + l)]; }
    double dcoeff(int n) const { return dc[static_cast<std::size_t>(n + l)]; }
};

// sin(pi x) / (pi x) and its derivative (sinc.hpp:15-36): c_0 and c_0' of the order x.
inline double sinc(double x) {
    double c[3], dc[3];
    detail::throw_status(fgfrft_sinc_coeffs(x, 1, c, dc));
    return c[1];
}
inline double sinc_deriv(double x) {
    double c[3], dc[3];
    detail::throw_status(fgfrft_sinc_coeffs(x, 1, c, dc));
    return dc[1];
}

inline SincCoeffs sinc_coeffs(double alpha, int l) {
    if (l < 1) throw parameter_error("sinc_coeffs: truncation order must be >= 1");
    SincCoeffs s;
    s.alpha = alpha;
    s.l = l;
    s.c.resize(2 * static_cast<std::size_t>(l) + 1);
    s.dc.resize(2 * static_cast<std::size_t>(l) + 1);
    detail::throw_status(fgfrft_sinc_coeffs(alpha, l, s.c.data(), s.dc.data()));
    return s;
}

}  // namespace fgfrft
#endif
