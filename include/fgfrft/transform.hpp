#pragma once
// Drop-in replacement for proj/include/fgfrft/transform.hpp (the FGFRFT hot path) backed by
// libfgfrft_b200.so: the power cache lives in B200 HBM, synthesis / apply / gradients run as
// hand-written sm_100a kernels. Names, signatures, error types and warning text follow the
// reference (transform.hpp:17-148); every divergence is listed here:
//   * PowerCache owns device memory: it is movable; copying re-uploads the powers (deep copy,
//     as the reference's implicit copy), and power(k) returns the matrix by value (one D2H copy).
//   * Constructor takes two optional trailing arguments (device, dtype) -- additive.
//   * Extensions (additive): fgfrft_matrices (many orders per launch), apply_series (F^a X
//     without a host round trip of F^a), order_gradient (sum_k c'_k Re<G, F^k X>).

#include <cmath>
#include <complex>
#include <cstdint>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "fgfrft/errors.hpp"
#include "fgfrft/gft.hpp"
#include "fgfrft/matrix.hpp"
#include "fgfrft/sinc.hpp"

namespace fgfrft {

inline constexpr std::uint64_t kDefaultMemoryBudget = 4ULL << 30;  // transform.hpp:17

// P_n = F^n, n = 1..L, resident on the GPU (transform.hpp:41-80).
class PowerCache {
  public:
    PowerCache(const GftMatrix& f, int l, std::uint64_t memory_budget = kDefaultMemoryBudget, int device = 0,
               fgfrft_dtype dtype = FGFRFT_C128) {
        if (l < 1) throw parameter_error("PowerCache: truncation order must be >= 1");
        if (f.f.rows() != f.f.cols()) throw shape_error("PowerCache: F must be square");
        detail::throw_status(fgfrft_cache_create(reinterpret_cast<const double*>(f.f.data()), f.f.rows(), l,
                                                 memory_budget, dtype, device, &h_));
        load_info();
    }

    PowerCache(const PowerCache& o) : budget_(o.budget_) {
        const Index n = o.n();
        std::vector<std::complex<double>> all(static_cast<size_t>(n * n * o.l_));
        for (int k = 1; k <= o.l_; ++k)
            detail::throw_status(fgfrft_cache_power(o.h_, k, reinterpret_cast<double*>(all.data() + (k - 1) * n * n)));
        int dtype = 0, device = 0;
        fgfrft_cache_info(o.h_, nullptr, nullptr, nullptr, &dtype, &device);
        detail::throw_status(fgfrft_cache_create_from_powers(reinterpret_cast<const double*>(all.data()),
                                                             reinterpret_cast<const double*>(all.data()), n, o.l_,
                                                             ~0ULL, dtype, device, &h_));
        load_info();
    }
    PowerCache(PowerCache&& o) noexcept : h_(std::exchange(o.h_, nullptr)), l_(o.l_), n_(o.n_), fp_(o.fp_) {}
    PowerCache& operator=(PowerCache o) noexcept {
        std::swap(h_, o.h_);
        l_ = o.l_;
        n_ = o.n_;
        fp_ = o.fp_;
        return *this;
    }
    ~PowerCache() {
        if (h_) fgfrft_cache_destroy(h_);
    }

    int l() const { return l_; }
    Index n() const { return n_; }
    std::uint64_t fingerprint() const { return fp_; }

    // F^k for k = 1..L (transform.hpp:131-134), copied to the host.
    MatrixXcd power(int k) const {
        if (k < 1 || k > l_) throw parameter_error("PowerCache: power index out of range");
        MatrixXcd out(n_, n_);
        detail::throw_status(fgfrft_cache_power(h_, k, reinterpret_cast<double*>(out.data())));
        return out;
    }

    void verify(const GftMatrix& f) const {  // transform.hpp:136-139
        if (content_fingerprint(f.f) != fp_)
            throw numerical_error("PowerCache: fingerprint mismatch, cache is stale for this matrix");
    }

    fgfrft_cache* handle() const { return h_; }

    // Extension: GEMM engine (FGFRFT_ENGINE_AUTO / _DMMA / _INT8, see fgfrft_b200.h) and eager
    // construction of the INT8 digit slices used by order sweeps on a real F.
    void set_engine(int engine) { detail::throw_status(fgfrft_cache_set_engine(h_, engine)); }
    void prepare() { detail::throw_status(fgfrft_cache_prepare(h_)); }

    // Extension: persist F and the resident powers; load() restores the
    // cache without the O(L n^3) recursion (io_error / parse_error / capacity_error /
    // numerical_error on a missing, malformed, over-budget or corrupt file).
    void save(const std::string& path) const { detail::throw_status(fgfrft_cache_save(h_, path.c_str())); }
    static PowerCache load(const std::string& path, std::uint64_t memory_budget = kDefaultMemoryBudget,
                           int device = 0) {
        fgfrft_cache* h = nullptr;
        detail::throw_status(fgfrft_cache_load(path.c_str(), memory_budget, device, &h));
        return PowerCache(h, memory_budget);
    }

  private:
    PowerCache(fgfrft_cache* h, std::uint64_t budget) : h_(h), budget_(budget) { load_info(); }
    void load_info() {
        int64_t n = 0;
        detail::throw_status(fgfrft_cache_info(h_, &n, &l_, &fp_, nullptr, nullptr));
        n_ = static_cast<Index>(n);
    }
    fgfrft_cache* h_ = nullptr;
    int l_ = 0;
    Index n_ = 0;
    std::uint64_t fp_ = 0;
    std::uint64_t budget_ = kDefaultMemoryBudget;
};

inline PowerCache build_power_cache(const GftMatrix& f, int l, std::uint64_t memory_budget = kDefaultMemoryBudget) {
    return PowerCache(f, l, memory_budget);
}

// Truncated-series operator (l >= 1) or exact spectral operator (l == 0), transform.hpp:89-93.
struct FracOperator {
    MatrixXcd q;
    double alpha = 0.0;
    int l = 0;
};

namespace detail {

inline void warn_if_outside_window(double alpha, int l) {  // transform.hpp:97-104
    if (std::fabs(alpha) > static_cast<double>(l) + 1.0) {
        std::ostringstream msg;
        msg << "order alpha = " << alpha << " lies outside the series window [-" << l + 1 << ", " << l + 1
            << "]; coefficient mass concentrates in dropped terms";
        warn(msg.str());
    }
}

inline int resolve_truncation(const PowerCache& cache, int truncation) {
    const int l = truncation == 0 ? cache.l() : truncation;
    if (l < 1 || l > cache.l()) throw parameter_error("fgfrft_matrix: truncation exceeds the cached power set");
    return l;
}

}  // namespace detail

// Q = c_0 I + sum_{n=1..L} [c_n F^n + c_{-n} (F^n)^H]  (transform.hpp:111-123).
inline FracOperator fgfrft_matrix(const PowerCache& cache, double alpha, int truncation = 0) {
    const int l = detail::resolve_truncation(cache, truncation);
    detail::warn_if_outside_window(alpha, l);
    FracOperator op{MatrixXcd(cache.n(), cache.n()), alpha, l};
    detail::throw_status(
        fgfrft_synthesize(cache.handle(), &alpha, 1, truncation, FGFRFT_Q, reinterpret_cast<double*>(op.q.data())));
    return op;
}

// dQ/dalpha from the same powers with c'_n (transform.hpp:127-136).
inline MatrixXcd fgfrft_grad(const PowerCache& cache, double alpha) {
    detail::warn_if_outside_window(alpha, cache.l());
    MatrixXcd g(cache.n(), cache.n());
    detail::throw_status(fgfrft_synthesize(cache.handle(), &alpha, 1, 0, FGFRFT_DQ, reinterpret_cast<double*>(g.data())));
    return g;
}

// Y = Q X (transform.hpp:138-141) on the DMMA GEMM.
inline MatrixXcd apply_forward(const FracOperator& op, const MatrixXcd& x) {
    if (x.rows() != op.q.cols()) throw shape_error("apply_forward: signal length does not match operator");
    MatrixXcd y(x.rows(), x.cols());
    detail::throw_status(fgfrft_apply_matrix(reinterpret_cast<const double*>(op.q.data()), op.q.rows(), 0,
                                             reinterpret_cast<const double*>(x.data()), x.cols(),
                                             reinterpret_cast<double*>(y.data()), 0));
    return y;
}

// Y = Q^H X = Q^{-alpha} X (transform.hpp:145-148).
inline MatrixXcd apply_inverse(const FracOperator& op, const MatrixXcd& x) {
    if (x.rows() != op.q.rows()) throw shape_error("apply_inverse: signal length does not match operator");
    MatrixXcd y(x.rows(), x.cols());
    detail::throw_status(fgfrft_apply_matrix(reinterpret_cast<const double*>(op.q.data()), op.q.rows(), 1,
                                             reinterpret_cast<const double*>(x.data()), x.cols(),
                                             reinterpret_cast<double*>(y.data()), 0));
    return y;
}

// ---- extensions ---------------------------------------------------------------------------

// Many orders in one launch (each cache tile crosses HBM once for the whole set).
inline std::vector<MatrixXcd> fgfrft_matrices(const PowerCache& cache, const std::vector<double>& alphas,
                                              int truncation = 0) {
    const int l = detail::resolve_truncation(cache, truncation);
    for (double a : alphas) detail::warn_if_outside_window(a, l);
    const Index n = cache.n();
    std::vector<std::complex<double>> buf(static_cast<size_t>(n * n) * alphas.size());
    detail::throw_status(fgfrft_synthesize(cache.handle(), alphas.data(), static_cast<int>(alphas.size()), truncation,
                                           FGFRFT_Q, reinterpret_cast<double*>(buf.data())));
    std::vector<MatrixXcd> out;
    for (size_t a = 0; a < alphas.size(); ++a) {
        MatrixXcd q(n, n);
        std::copy(buf.begin() + static_cast<std::ptrdiff_t>(a * n * n),
                  buf.begin() + static_cast<std::ptrdiff_t>((a + 1) * n * n), q.data());
        out.push_back(std::move(q));
    }
    return out;
}

// F^alpha X (or (F^alpha)^H X) with F^alpha synthesised and consumed on the device.
inline MatrixXcd apply_series(const PowerCache& cache, double alpha, const MatrixXcd& x, bool inverse = false,
                              int truncation = 0) {
    if (x.rows() != cache.n()) throw shape_error("apply_forward: signal length does not match operator");
    const int l = detail::resolve_truncation(cache, truncation);
    detail::warn_if_outside_window(alpha, l);
    MatrixXcd y(x.rows(), x.cols());
    detail::throw_status(fgfrft_apply(cache.handle(), &alpha, 1, truncation, inverse ? 1 : 0,
                                      reinterpret_cast<const double*>(x.data()), x.cols(),
                                      reinterpret_cast<double*>(y.data())));
    return y;
}

// dL/dalpha = sum_k c'_k(alpha) Re<G, F^k X> (learn.hpp:88-92 contraction); s (optional)
// receives the 2L+1 per-power terms in SincCoeffs layout.
inline double order_gradient(const PowerCache& cache, double alpha, const MatrixXcd& g, const MatrixXcd& x,
                             std::vector<double>* s = nullptr) {
    if (x.rows() != cache.n() || g.rows() != x.rows() || g.cols() != x.cols())
        throw shape_error("order_gradient: cotangent / signal shape mismatch");
    std::vector<double> terms(2 * static_cast<size_t>(cache.l()) + 1);
    double out = 0.0;
    detail::throw_status(fgfrft_dlda(cache.handle(), &alpha, 1, reinterpret_cast<const double*>(g.data()),
                                     reinterpret_cast<const double*>(x.data()), x.cols(), terms.data(), &out));
    if (s) *s = std::move(terms);
    return out;
}

}  // namespace fgfrft
