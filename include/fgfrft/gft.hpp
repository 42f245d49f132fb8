#pragma once
// GFT matrices (reference: proj/include/fgfrft/gft.hpp). The drop-in replaces only the hot path
// (transform.hpp, spectral.hpp, learn.hpp); with the reference headers on the include path (Eigen
// builds, include/ before proj/include) this header forwards to the reference's own gft.hpp, so
// GftMatrix, gft_from_shift, random_unitary, synthetic_unitary and unitarity_residual are the
// reference's. Without Eigen it provides the same names and semantics on the minimal matrix type:
// gft_from_shift by a cyclic Jacobi eigensolver followed by the reference's post-processing
// (ascending eigenvalues, modified Gram-Schmidt inside degenerate clusters, sign pivot = first
// largest |component| made positive, cluster columns ordered by pivot; gft.hpp:74-128), and
// random_unitary by a Householder QR with the R diagonal phases divided out (unique, so equal to
// the reference's up to rounding). F itself is input preparation, not the hot path.
#include "fgfrft/matrix.hpp"

#if defined(FGFRFT_HAVE_EIGEN) && __has_include_next(<fgfrft/gft.hpp>)
#include_next <fgfrft/gft.hpp>
#else
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <optional>
#include <sstream>
#include <utility>
#include <vector>

#include "fgfrft/errors.hpp"
#include "fgfrft/graph.hpp"
#include "fgfrft/rng.hpp"

namespace fgfrft {

enum class Provenance { graph, haar, synthetic };

// Eigenbasis and eigenphases recorded at construction time (gft.hpp:21-25).
struct KnownSpectrum {
    MatrixXcd v;     // unitary eigenvector matrix
    VectorXd theta;  // phases in (-pi, pi)
};

struct GftMatrix {
    MatrixXcd f;
    Provenance provenance = Provenance::graph;
    std::optional<KnownSpectrum> known_spectrum;

    Index n() const { return f.rows(); }

    bool is_real(double tol = 1e-13) const {
        for (Index j = 0; j < f.cols(); ++j)
            for (Index i = 0; i < f.rows(); ++i)
                if (std::abs(f(i, j).imag()) > tol) return false;
        return true;
    }
};

// ||F F^H - I||_F / sqrt(n) (gft.hpp:39-44).
inline double unitarity_residual(const MatrixXcd& f) {
    const Index n = f.rows();
    double s = 0.0;
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) {
            std::complex<double> g = 0.0;
            for (Index k = 0; k < f.cols(); ++k) g += f(i, k) * std::conj(f(j, k));
            if (i == j) g -= 1.0;
            s += std::norm(g);
        }
    return std::sqrt(s) / std::sqrt(static_cast<double>(n));
}

inline std::uint64_t content_fingerprint(const MatrixXcd& m) {
    return fgfrft_fnv1a64(m.data(), sizeof(std::complex<double>) * static_cast<size_t>(m.rows() * m.cols()));
}

namespace detail {

// Cyclic Jacobi eigensolver of a real symmetric matrix: eigenvalues (unsorted) and eigenvectors
// in the columns of v. Converges quadratically; O(n^3) per sweep (a small-graph fallback).
inline void jacobi_eigen(MatrixXd a, std::vector<double>& lambda, MatrixXd& v) {
    const Index n = a.rows();
    v = MatrixXd::Zero(n, n);
    for (Index i = 0; i < n; ++i) v(i, i) = 1.0;
    const double total = std::max(a.norm(), 1e-300);
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0.0;
        for (Index q = 0; q < n; ++q)
            for (Index p = 0; p < q; ++p) off += a(p, q) * a(p, q);
        if (std::sqrt(2.0 * off) <= 1e-15 * total) break;
        for (Index q = 1; q < n; ++q)
            for (Index p = 0; p < q; ++p) {
                const double apq = a(p, q);
                if (apq == 0.0) continue;
                const double theta = (a(q, q) - a(p, p)) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (Index k = 0; k < n; ++k) {  // A <- J^T A J, columns then rows
                    const double akp = a(k, p), akq = a(k, q);
                    a(k, p) = c * akp - s * akq;
                    a(k, q) = s * akp + c * akq;
                }
                for (Index k = 0; k < n; ++k) {
                    const double apk = a(p, k), aqk = a(q, k);
                    a(p, k) = c * apk - s * aqk;
                    a(q, k) = s * apk + c * aqk;
                }
                for (Index k = 0; k < n; ++k) {
                    const double vkp = v(k, p), vkq = v(k, q);
                    v(k, p) = c * vkp - s * vkq;
                    v(k, q) = s * vkp + c * vkq;
                }
            }
    }
    lambda.resize(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) lambda[static_cast<size_t>(i)] = a(i, i);
}

inline Index sign_pivot_col(const MatrixXd& v, Index col) {  // first component of largest |value|
    Index p = 0;
    double best = std::fabs(v(0, col));
    for (Index i = 1; i < v.rows(); ++i)
        if (std::fabs(v(i, col)) > best) {
            best = std::fabs(v(i, col));
            p = i;
        }
    return p;
}

}  // namespace detail

// F = V^T for Z = V diag(lambda) V^T, ascending lambda, deterministic signs (gft.hpp:74-128).
inline GftMatrix gft_from_shift(const ShiftOperator& z) {
    const Index n = z.matrix.rows();
    if (n != z.matrix.cols()) throw shape_error("gft_from_shift: shift operator must be square");
    double asym = 0.0;
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) {
            const double d = z.matrix(i, j) - z.matrix(j, i);
            asym += d * d;
        }
    if (std::sqrt(asym) > 1e-12 * std::max(1.0, z.matrix.norm()))
        throw numerical_error("gft_from_shift: shift operator is not symmetric");
    std::vector<double> lam;
    MatrixXd vr;
    detail::jacobi_eigen(z.matrix, lam, vr);
    std::vector<Index> order(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) order[static_cast<size_t>(i)] = i;
    std::stable_sort(order.begin(), order.end(), [&](Index a, Index b) { return lam[a] < lam[b]; });
    MatrixXd v(n, n);
    std::vector<double> lambda(static_cast<size_t>(n));
    for (Index c = 0; c < n; ++c) {
        lambda[static_cast<size_t>(c)] = lam[order[static_cast<size_t>(c)]];
        for (Index i = 0; i < n; ++i) v(i, c) = vr(i, order[static_cast<size_t>(c)]);
    }
    const double scale = std::max(1.0, std::max(std::fabs(lambda.front()), std::fabs(lambda.back())));
    const double cluster_tol = 1e-9 * scale;
    Index lo = 0;
    while (lo < n) {
        Index hi = lo;
        while (hi + 1 < n && lambda[static_cast<size_t>(hi + 1)] - lambda[static_cast<size_t>(hi)] <= cluster_tol) ++hi;
        const Index k = hi - lo + 1;
        if (k > 1)  // modified Gram-Schmidt inside the cluster
            for (Index a = 0; a < k; ++a) {
                for (Index b = 0; b < a; ++b) {
                    double d = 0.0;
                    for (Index i = 0; i < n; ++i) d += v(i, lo + b) * v(i, lo + a);
                    for (Index i = 0; i < n; ++i) v(i, lo + a) -= d * v(i, lo + b);
                }
                double nr = 0.0;
                for (Index i = 0; i < n; ++i) nr += v(i, lo + a) * v(i, lo + a);
                nr = std::sqrt(nr);
                for (Index i = 0; i < n; ++i) v(i, lo + a) /= nr;
            }
        std::vector<std::pair<Index, Index>> piv;  // (pivot, column)
        for (Index a = lo; a <= hi; ++a) {
            const Index p = detail::sign_pivot_col(v, a);
            if (v(p, a) < 0.0)
                for (Index i = 0; i < n; ++i) v(i, a) = -v(i, a);
            piv.emplace_back(p, a);
        }
        if (k > 1) {
            std::sort(piv.begin(), piv.end());
            MatrixXd block(n, k);
            for (Index a = 0; a < k; ++a)
                for (Index i = 0; i < n; ++i) block(i, a) = v(i, piv[static_cast<size_t>(a)].second);
            for (Index a = 0; a < k; ++a)
                for (Index i = 0; i < n; ++i) v(i, lo + a) = block(i, a);
        }
        lo = hi + 1;
    }
    GftMatrix out;
    out.provenance = Provenance::graph;
    out.f = MatrixXcd(n, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) out.f(i, j) = v(j, i);
    const double resid = unitarity_residual(out.f);
    if (resid > 1e-10) {
        std::ostringstream msg;
        msg << "gft_from_shift: unitarity residual " << resid << " exceeds 1e-10";
        throw numerical_error(msg.str());
    }
    return out;
}

// Haar unitary: QR of a complex Gaussian matrix (entries (g, g) / sqrt 2 in column-major order of
// the Rng stream), R's diagonal phases divided out -- Q with a positive real R diagonal.
inline GftMatrix random_unitary(Index n, std::uint64_t seed) {
    if (n < 1) throw parameter_error("random_unitary: n must be >= 1");
    Rng rng(seed);
    MatrixXcd a(n, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) {
            const double re = rng.gaussian(), im = rng.gaussian();
            a(i, j) = std::complex<double>(re, im) * M_SQRT1_2;
        }
    // Householder QR: reflectors v_k (stored), R in a's upper triangle
    std::vector<std::vector<std::complex<double>>> refl(static_cast<size_t>(n));
    std::vector<std::complex<double>> rdiag(static_cast<size_t>(n));
    for (Index k = 0; k < n; ++k) {
        double xn = 0.0;
        for (Index i = k; i < n; ++i) xn += std::norm(a(i, k));
        xn = std::sqrt(xn);
        const std::complex<double> x0 = a(k, k);
        const std::complex<double> ph = std::abs(x0) > 0.0 ? x0 / std::abs(x0) : std::complex<double>(1.0, 0.0);
        const std::complex<double> alpha = -ph * xn;
        std::vector<std::complex<double>> v(static_cast<size_t>(n - k));
        for (Index i = k; i < n; ++i) v[static_cast<size_t>(i - k)] = a(i, k);
        v[0] -= alpha;
        double vn = 0.0;
        for (const auto& e : v) vn += std::norm(e);
        vn = std::sqrt(vn);
        if (vn > 0.0)
            for (auto& e : v) e /= vn;
        for (Index j = k; j < n; ++j) {  // A <- (I - 2 v v^H) A
            std::complex<double> d = 0.0;
            for (Index i = k; i < n; ++i) d += std::conj(v[static_cast<size_t>(i - k)]) * a(i, j);
            for (Index i = k; i < n; ++i) a(i, j) -= 2.0 * v[static_cast<size_t>(i - k)] * d;
        }
        rdiag[static_cast<size_t>(k)] = a(k, k);
        refl[static_cast<size_t>(k)] = std::move(v);
    }
    MatrixXcd q = MatrixXcd::Identity(n, n);  // Q = H_0 H_1 ... H_(n-1), applied right to left
    for (Index k = n - 1; k >= 0; --k) {
        const auto& v = refl[static_cast<size_t>(k)];
        for (Index j = 0; j < n; ++j) {
            std::complex<double> d = 0.0;
            for (Index i = k; i < n; ++i) d += std::conj(v[static_cast<size_t>(i - k)]) * q(i, j);
            for (Index i = k; i < n; ++i) q(i, j) -= 2.0 * v[static_cast<size_t>(i - k)] * d;
        }
    }
    GftMatrix out;
    out.provenance = Provenance::haar;
    out.f = MatrixXcd(n, n);
    for (Index k = 0; k < n; ++k) {
        const std::complex<double> d = rdiag[static_cast<size_t>(k)];
        const double m = std::abs(d);
        const std::complex<double> p = m > 0.0 ? d / m : std::complex<double>(1.0, 0.0);
        for (Index i = 0; i < n; ++i) out.f(i, k) = q(i, k) * p;
    }
    return out;
}

// F = V diag(e^{j theta}) V^H over a Haar basis V; the spectrum is recorded (gft.hpp:159-177).
inline GftMatrix synthetic_unitary(const std::vector<double>& phases, std::uint64_t seed) {
    const Index n = static_cast<Index>(phases.size());
    if (n < 1) throw parameter_error("synthetic_unitary: need at least one phase");
    for (double t : phases)
        if (!(std::fabs(t) < M_PI)) throw parameter_error("synthetic_unitary: phases must satisfy |theta| < pi");
    GftMatrix basis = random_unitary(n, seed);
    VectorXd theta(n);
    MatrixXcd scaled(n, n);
    for (Index k = 0; k < n; ++k) {
        theta(k) = phases[static_cast<size_t>(k)];
        const std::complex<double> e = std::polar(1.0, theta(k));
        for (Index i = 0; i < n; ++i) scaled(i, k) = basis.f(i, k) * e;
    }
    GftMatrix out;
    out.provenance = Provenance::synthetic;
    out.f = scaled * basis.f.adjoint();
    out.known_spectrum = KnownSpectrum{std::move(basis.f), std::move(theta)};
    return out;
}

}  // namespace fgfrft
#endif
