#pragma once
// Drop-in replacement for proj/include/fgfrft/spectral.hpp backed by libfgfrft_b200.so: the
// eigendecomposition of a unitary F runs its Hermitian stage on cuSOLVER and its products on the
// GPU, the exact fractional power F^a = V diag(e^{j a theta}) V^H is one FP64 tensor-core GEMM.
// Same names and semantics (spectral.hpp:19-195); divergences:
//   * UnitaryEigen additionally carries a shared handle to its device copy (V stays in HBM).
//   * Eigenvector phases / the basis inside an eigenvalue cluster may differ from Eigen's (the
//     decomposition is unique only up to those); operators built from it agree to rounding.

#include <cmath>
#include <memory>
#include <sstream>
#include <vector>

#include "fgfrft/errors.hpp"
#include "fgfrft/gft.hpp"
#include "fgfrft/matrix.hpp"
#include "fgfrft/transform.hpp"

namespace fgfrft {

struct UnitaryEigen {  // spectral.hpp:19-31
    MatrixXcd v;
    VectorXd theta;  // ascending in (-pi, pi]

    Index n() const { return v.rows(); }

    std::vector<std::complex<double>> eigenvalues() const {
        std::vector<std::complex<double>> lam(static_cast<size_t>(theta.size()));
        for (Index k = 0; k < theta.size(); ++k) lam[static_cast<size_t>(k)] = std::polar(1.0, theta(k));
        return lam;
    }

    // Device copy (created on first use from v / theta when the spectrum was built on the host).
    fgfrft_spectrum* device_handle(int device = 0) const {
        if (!dev_) {
            fgfrft_spectrum* h = nullptr;
            detail::throw_status(fgfrft_spectrum_create(reinterpret_cast<const double*>(v.data()), theta.data(),
                                                        v.rows(), device, &h));
            dev_.reset(h, [](fgfrft_spectrum* p) { fgfrft_spectrum_destroy(p); });
        }
        return dev_.get();
    }
    void adopt(fgfrft_spectrum* h) const { dev_.reset(h, [](fgfrft_spectrum* p) { fgfrft_spectrum_destroy(p); }); }

  private:
    mutable std::shared_ptr<fgfrft_spectrum> dev_;
};

// spectral.hpp:121-155. A recorded spectrum is returned as stored.
inline UnitaryEigen eigendecompose_unitary(const GftMatrix& f, int device = 0) {
    UnitaryEigen out;
    if (f.known_spectrum) {
        out.v = f.known_spectrum->v;
        out.theta = f.known_spectrum->theta;
        return out;
    }
    fgfrft_spectrum* h = nullptr;
    detail::throw_status(fgfrft_spectrum_decompose(reinterpret_cast<const double*>(f.f.data()), f.n(), device, &h));
    out.adopt(h);
    const Index n = f.n();
    out.v = MatrixXcd(n, n);
    out.theta = VectorXd(n);
    detail::throw_status(fgfrft_spectrum_info(h, nullptr, out.theta.data()));
    detail::throw_status(fgfrft_spectrum_vectors(h, reinterpret_cast<double*>(out.v.data())));
    return out;
}

// Exact fractional power F^alpha = V diag(e^{j alpha theta}) V^H (spectral.hpp:158-166).
inline FracOperator exact_gfrft(const UnitaryEigen& e, double alpha) {
    FracOperator op;
    op.alpha = alpha;
    op.l = 0;
    op.q = MatrixXcd(e.n(), e.n());
    detail::throw_status(
        fgfrft_exact(e.device_handle(), &alpha, 1, FGFRFT_Q, reinterpret_cast<double*>(op.q.data())));
    return op;
}

// d F^alpha / d alpha = V diag(j theta e^{j alpha theta}) V^H (spectral.hpp:169-174).
inline MatrixXcd exact_gfrft_grad(const UnitaryEigen& e, double alpha) {
    MatrixXcd g(e.n(), e.n());
    detail::throw_status(fgfrft_exact(e.device_handle(), &alpha, 1, FGFRFT_DQ, reinterpret_cast<double*>(g.data())));
    return g;
}

// min_k (pi - |theta_k|), warning below 0.05 pi (spectral.hpp:179-195).
inline double phase_margin(const GftMatrix& f) {
    VectorXd theta = f.known_spectrum ? f.known_spectrum->theta : eigendecompose_unitary(f).theta;
    double margin = M_PI;
    for (Index k = 0; k < theta.size(); ++k) margin = std::min(margin, M_PI - std::fabs(theta(k)));
    if (margin < 0.05 * M_PI) {
        std::ostringstream msg;
        msg << "phase margin " << margin << " is below 0.05*pi; series approximation accuracy is at risk";
        warn(msg.str());
    }
    return margin;
}

}  // namespace fgfrft
