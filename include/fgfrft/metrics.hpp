#pragma once
// Approximation-error triple (reference: proj/include/fgfrft/metrics.hpp:13-34). With the
// reference headers on the include path (Eigen builds) this forwards to the reference's header.
#include "fgfrft/matrix.hpp"

#if defined(FGFRFT_HAVE_EIGEN) && __has_include_next(<fgfrft/metrics.hpp>)
#include_next <fgfrft/metrics.hpp>
#else
#include <cmath>

#include "fgfrft/errors.hpp"

namespace fgfrft {

// Over D = approx - reference: MSE and MAE are element means, NMSE = ||D||_F^2 / ||reference||_F^2.
struct ErrorReport {
    double mse = 0.0;
    double mae = 0.0;
    double nmse = 0.0;
    Index n = 0;
};

inline ErrorReport matrix_errors(const MatrixXcd& approx, const MatrixXcd& reference) {
    if (approx.rows() != reference.rows() || approx.cols() != reference.cols())
        throw shape_error("matrix_errors: shape mismatch");
    const double ref_sq = reference.squaredNorm();
    if (ref_sq == 0.0) throw numerical_error("matrix_errors: NMSE undefined for all-zero reference");
    double sq = 0.0, ab = 0.0;
    for (Index j = 0; j < approx.cols(); ++j)
        for (Index i = 0; i < approx.rows(); ++i) {
            const auto d = approx(i, j) - reference(i, j);
            sq += std::norm(d);
            ab += std::abs(d);
        }
    const double count = static_cast<double>(approx.rows() * approx.cols());
    ErrorReport r;
    r.n = approx.rows();
    r.mse = sq / count;
    r.mae = ab / count;
    r.nmse = sq / ref_sq;
    return r;
}

}  // namespace fgfrft
#endif
