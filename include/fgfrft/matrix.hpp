#pragma once
// Dense complex matrix used at the drop-in boundary. With Eigen available the reference's own
// type is used (Eigen::MatrixXcd: column-major std::complex<double>); otherwise a minimal
// column-major matrix with the same data()/rows()/cols()/(i,j) contract stands in, so callers
// written against the reference compile against either.

#include <cmath>
#include <complex>
#include <cstdint>
#include <vector>

#if __has_include(<Eigen/Dense>) && !defined(FGFRFT_NO_EIGEN)
#include <Eigen/Dense>
namespace fgfrft {
using MatrixXcd = Eigen::MatrixXcd;
using VectorXd = Eigen::VectorXd;
using MatrixXd = Eigen::MatrixXd;
using Index = Eigen::Index;
}  // namespace fgfrft
#define FGFRFT_HAVE_EIGEN 1
#else
namespace fgfrft {

using Index = std::ptrdiff_t;

class MatrixXcd {
  public:
    using Scalar = std::complex<double>;
    MatrixXcd() = default;
    MatrixXcd(Index r, Index c) : r_(r), c_(c), d_(static_cast<size_t>(r * c)) {}

    static MatrixXcd Zero(Index r, Index c) { return MatrixXcd(r, c); }
    static MatrixXcd Identity(Index r, Index c) {
        MatrixXcd m(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
        return m;
    }

    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    Scalar* data() { return d_.data(); }
    const Scalar* data() const { return d_.data(); }
    Scalar& operator()(Index i, Index j) { return d_[static_cast<size_t>(i + j * r_)]; }
    const Scalar& operator()(Index i, Index j) const { return d_[static_cast<size_t>(i + j * r_)]; }
    Scalar& operator()(Index i) { return d_[static_cast<size_t>(i)]; }
    const Scalar& operator()(Index i) const { return d_[static_cast<size_t>(i)]; }
    void resize(Index r, Index c) {
        r_ = r;
        c_ = c;
        d_.assign(static_cast<size_t>(r * c), Scalar(0.0));
    }

    MatrixXcd adjoint() const {
        MatrixXcd t(c_, r_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) t(j, i) = std::conj((*this)(i, j));
        return t;
    }
    double squaredNorm() const {
        double s = 0.0;
        for (const auto& v : d_) s += std::norm(v);
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    double maxAbs() const {
        double m = 0.0;
        for (const auto& v : d_) m = std::max(m, std::abs(v));
        return m;
    }
    bool operator==(const MatrixXcd& o) const { return r_ == o.r_ && c_ == o.c_ && d_ == o.d_; }
    MatrixXcd operator-(const MatrixXcd& o) const {
        MatrixXcd m(r_, c_);
        for (size_t i = 0; i < d_.size(); ++i) m.d_[i] = d_[i] - o.d_[i];
        return m;
    }
    MatrixXcd operator+(const MatrixXcd& o) const {
        MatrixXcd m(r_, c_);
        for (size_t i = 0; i < d_.size(); ++i) m.d_[i] = d_[i] + o.d_[i];
        return m;
    }
    MatrixXcd operator*(double s) const {
        MatrixXcd m(*this);
        for (auto& v : m.d_) v *= s;
        return m;
    }
    // Host product for small test-side checks (the hot-path products run on the GPU).
    MatrixXcd operator*(const MatrixXcd& o) const {
        MatrixXcd m(r_, o.c_);
        for (Index j = 0; j < o.c_; ++j)
            for (Index k = 0; k < c_; ++k) {
                const Scalar b = o(k, j);
                for (Index i = 0; i < r_; ++i) m(i, j) += (*this)(i, k) * b;
            }
        return m;
    }

  private:
    Index r_ = 0, c_ = 0;
    std::vector<Scalar> d_;
};

// Real dense matrix (column-major) with the Eigen::MatrixXd members the graph / GFT fallbacks use.
class MatrixXd {
  public:
    using Scalar = double;
    MatrixXd() = default;
    MatrixXd(Index r, Index c) : r_(r), c_(c), d_(static_cast<size_t>(r * c), 0.0) {}
    static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    double* data() { return d_.data(); }
    const double* data() const { return d_.data(); }
    double& operator()(Index i, Index j) { return d_[static_cast<size_t>(i + j * r_)]; }
    const double& operator()(Index i, Index j) const { return d_[static_cast<size_t>(i + j * r_)]; }
    double squaredNorm() const {
        double s = 0.0;
        for (double v : d_) s += v * v;
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    MatrixXd transpose() const {
        MatrixXd t(c_, r_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
        return t;
    }

  private:
    Index r_ = 0, c_ = 0;
    std::vector<double> d_;
};

// Real vector with the Eigen::VectorXd members the learning API uses.
class VectorXd {
  public:
    VectorXd() = default;
    explicit VectorXd(Index n) : d_(static_cast<size_t>(n), 0.0) {}
    static VectorXd Zero(Index n) { return VectorXd(n); }
    static VectorXd Constant(Index n, double v) {
        VectorXd x(n);
        for (auto& e : x.d_) e = v;
        return x;
    }
    Index size() const { return static_cast<Index>(d_.size()); }
    double* data() { return d_.data(); }
    const double* data() const { return d_.data(); }
    double& operator()(Index i) { return d_[static_cast<size_t>(i)]; }
    const double& operator()(Index i) const { return d_[static_cast<size_t>(i)]; }
    double& operator[](Index i) { return d_[static_cast<size_t>(i)]; }
    const double& operator[](Index i) const { return d_[static_cast<size_t>(i)]; }
    void resize(Index n) { d_.assign(static_cast<size_t>(n), 0.0); }
    double sum() const {
        double s = 0.0;
        for (double v : d_) s += v;
        return s;
    }

  private:
    std::vector<double> d_;
};

}  // namespace fgfrft
#endif
