#pragma once
// Drop-in for the cascaded transform-order learning of proj/include/fgfrft/learn.hpp:25-166,
// backed by libfgfrft_b200.so: the layer operators (series synthesis from the device power cache,
// or the exact spectral form), the prefix products, the reverse gradient accumulation and the
// Adam loop run on the GPU (fgfrft_cascade_*). Same names, fields, error types and messages.
// Divergence: the denoising learner of learn.hpp:168-516 is exposed through the C ABI
// (fgfrft_denoise_*, real F, fast engine) rather than through DenoiseProblem here.

#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <optional>
#include <vector>

#include "fgfrft/errors.hpp"
#include "fgfrft/gft.hpp"
#include "fgfrft/matrix.hpp"
#include "fgfrft/spectral.hpp"
#include "fgfrft/transform.hpp"

namespace fgfrft {

enum class Backend { exact, fast };

inline const char* backend_name(Backend b) { return b == Backend::exact ? "exact" : "fast"; }

struct CascadeConfig {  // learn.hpp:33-50
    int depth = 1;
    double init_order = 0.1;
    double target_order = 1.5;
    int truncation = 10;
    int epochs = 200;
    double lr = 0.01;
    std::uint64_t seed = 0;
    std::uint64_t memory_budget = kDefaultMemoryBudget;

    void validate() const {
        if (depth < 1) throw parameter_error("CascadeConfig: depth must be >= 1");
        if (epochs < 1) throw parameter_error("CascadeConfig: epochs must be >= 1");
        if (truncation < 1) throw parameter_error("CascadeConfig: truncation must be >= 1");
        if (!(lr > 0.0)) throw parameter_error("CascadeConfig: lr must be positive");
    }
};

// learn.hpp:52-116: loss and per-layer order gradients of the cascade (X = I, exact target).
class CascadeProblem {
  public:
    CascadeProblem(const GftMatrix& f, const CascadeConfig& cfg, Backend backend, int device = 0)
        : backend_(backend), cfg_(cfg) {
        cfg_.validate();
        n_ = f.n();
        eig_ = eigendecompose_unitary(f, device);
        if (backend_ == Backend::fast) cache_.emplace(f, cfg_.truncation, cfg_.memory_budget, device);
        fgfrft_cascade* h = nullptr;
        detail::throw_status(fgfrft_cascade_create(cache_ ? cache_->handle() : nullptr, eig_.device_handle(device),
                                                   cfg_.target_order, cfg_.depth, &h));
        h_.reset(h, [](fgfrft_cascade* p) { fgfrft_cascade_destroy(p); });
    }

    struct Eval {
        double loss = 0.0;
        VectorXd grad;
    };

    Eval eval(const VectorXd& alphas) const {
        if (alphas.size() != cfg_.depth) throw shape_error("CascadeProblem: one order per layer");
        Eval out;
        out.grad = VectorXd(alphas.size());
        detail::throw_status(fgfrft_cascade_eval(h_.get(), alphas.data(), &out.loss, out.grad.data()));
        return out;
    }

    Index n() const { return n_; }
    fgfrft_cascade* handle() const { return h_.get(); }

  private:
    Backend backend_;
    CascadeConfig cfg_;
    Index n_ = 0;
    UnitaryEigen eig_;
    std::optional<PowerCache> cache_;
    std::shared_ptr<fgfrft_cascade> h_;
};

struct OrderTrajectoryPoint {  // learn.hpp:118-123
    int epoch = 0;
    double loss = 0.0;
    std::vector<double> alphas;
    double alpha_sum = 0.0;
};

struct OrderLearnResult {  // learn.hpp:125-130
    std::vector<OrderTrajectoryPoint> trajectory;
    double final_loss = 0.0;
    std::vector<double> final_alphas;
    double final_alpha_sum = 0.0;
};

// learn.hpp:132-166: Adam from init_order, one record per epoch plus the final point.
inline OrderLearnResult learn_orders(const GftMatrix& f, const CascadeConfig& cfg, Backend backend, int device = 0) {
    cfg.validate();
    const CascadeProblem problem(f, cfg, backend, device);
    const int k = cfg.depth, e = cfg.epochs;
    std::vector<double> tl(static_cast<size_t>(e + 1)), ta(static_cast<size_t>(e + 1) * k), fa(static_cast<size_t>(k));
    OrderLearnResult out;
    detail::throw_status(fgfrft_cascade_learn(problem.handle(), cfg.init_order, e, cfg.lr, tl.data(), ta.data(),
                                              &out.final_loss, fa.data()));
    out.trajectory.reserve(static_cast<size_t>(e + 1));
    for (int i = 0; i <= e; ++i) {
        OrderTrajectoryPoint p;
        p.epoch = i;
        p.loss = tl[static_cast<size_t>(i)];
        p.alphas.assign(ta.begin() + static_cast<std::ptrdiff_t>(i) * k, ta.begin() + static_cast<std::ptrdiff_t>(i + 1) * k);
        for (double a : p.alphas) p.alpha_sum += a;
        out.trajectory.push_back(std::move(p));
    }
    out.final_alphas = fa;
    for (double a : fa) out.final_alpha_sum += a;
    return out;
}

// ---------------------------------------------------------------------------------------------
// Joint order/filter denoising (learn.hpp:168-516)

struct DenoiseConfig {  // learn.hpp:168-184
    int truncation = 10;
    int epochs = 300;
    double lr = 0.01;
    double init_alpha = 0.5;
    double sigma = 0.0;
    std::uint64_t seed = 0;
    bool loss_on_real = false;

    void validate() const {
        if (truncation < 1) throw parameter_error("DenoiseConfig: truncation must be >= 1");
        if (epochs < 1) throw parameter_error("DenoiseConfig: epochs must be >= 1");
        if (!(lr > 0.0)) throw parameter_error("DenoiseConfig: lr must be positive");
        if (sigma < 0.0) throw parameter_error("DenoiseConfig: sigma must be >= 0");
    }
};

struct FilterDiag {
    VectorXd h;
};

namespace detail {
struct DenoiseEval {
    double loss = 0.0;
    double grad_alpha = 0.0;
    VectorXd grad_h;
};
}  // namespace detail

// Real n x C matrix at the denoising boundary (Eigen::MatrixXd when Eigen is present).
#ifdef FGFRFT_HAVE_EIGEN
using MatrixXdN = Eigen::MatrixXd;
#else
struct MatrixXdN {
    MatrixXdN() = default;
    MatrixXdN(Index r, Index c) : r_(r), c_(c), d_(static_cast<size_t>(r * c), 0.0) {}
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    double* data() { return d_.data(); }
    const double* data() const { return d_.data(); }
    double& operator()(Index i, Index j) { return d_[static_cast<size_t>(i + j * r_)]; }
    const double& operator()(Index i, Index j) const { return d_[static_cast<size_t>(i + j * r_)]; }

  private:
    Index r_ = 0, c_ = 0;
    std::vector<double> d_;
};
#endif

class DenoiseProblem {  // learn.hpp:439-467
  public:
    DenoiseProblem(const MatrixXdN& y, const MatrixXdN& x_ref, const GftMatrix& f, const DenoiseConfig& cfg,
                   Backend backend, std::shared_ptr<const UnitaryEigen> spectrum = nullptr, int device = 0)
        : n_(f.n()), ch_(y.cols()) {
        cfg.validate();
        if (y.rows() != x_ref.rows() || y.cols() != x_ref.cols())
            throw shape_error("denoise: noisy and reference signals have mismatched channels");
        if (y.rows() != f.n()) throw shape_error("denoise: signal length does not match the graph");
        fgfrft_denoise* h = nullptr;
        if (backend == Backend::exact) {
            if (!spectrum) spectrum = std::make_shared<UnitaryEigen>(eigendecompose_unitary(f, device));
            spec_ = spectrum;
            detail::throw_status(fgfrft_denoise_create_exact(spectrum->device_handle(device), y.data(), x_ref.data(),
                                                             ch_, cfg.loss_on_real ? 1 : 0, &h));
        } else {
            cache_.emplace(f, cfg.truncation, std::uint64_t(1) << 40, device);
            detail::throw_status(fgfrft_denoise_create_ex(cache_->handle(), y.data(), x_ref.data(), ch_,
                                                          cfg.loss_on_real ? 1 : 0, &h));
        }
        h_.reset(h, [](fgfrft_denoise* p) { fgfrft_denoise_destroy(p); });
    }

    detail::DenoiseEval eval(double alpha, const VectorXd& h) const {
        detail::DenoiseEval out;
        out.grad_h = VectorXd(n_);
        detail::throw_status(fgfrft_denoise_eval(h_.get(), alpha, h.data(), &out.loss, &out.grad_alpha,
                                                 out.grad_h.data()));
        return out;
    }
    MatrixXdN reconstruct(double alpha, const VectorXd& h) const {
        MatrixXdN out(n_, ch_);
        detail::throw_status(fgfrft_denoise_reconstruct(h_.get(), alpha, h.data(), out.data()));
        return out;
    }
    Index n() const { return n_; }
    fgfrft_denoise* handle() const { return h_.get(); }
    Index channels() const { return ch_; }

  private:
    Index n_ = 0, ch_ = 0;
    std::optional<PowerCache> cache_;
    std::shared_ptr<const UnitaryEigen> spec_;
    std::shared_ptr<fgfrft_denoise> h_;
};

struct DenoiseTrajectoryPoint {
    int epoch = 0;
    double loss = 0.0;
    double alpha = 0.0;
};

struct DenoiseResult {  // learn.hpp:423-430
    double alpha_best = 0.0;
    FilterDiag filter_best;
    MatrixXdN reconstruction;
    std::vector<DenoiseTrajectoryPoint> trajectory;
    double loss_best = 0.0;
    int best_epoch = 0;
};

// learn.hpp:470-516: Adam over [alpha, h] from [init_alpha, 1..1] on the device.
inline DenoiseResult denoise(const MatrixXdN& y, const MatrixXdN& x_ref, const GftMatrix& f, const DenoiseConfig& cfg,
                             Backend backend, std::shared_ptr<const UnitaryEigen> spectrum = nullptr,
                             int device = 0) {
    cfg.validate();
    const DenoiseProblem problem(y, x_ref, f, cfg, backend, std::move(spectrum), device);
    const Index n = f.n();
    const int e = cfg.epochs;
    std::vector<double> tl(static_cast<size_t>(e + 1)), ta(static_cast<size_t>(e + 1));
    DenoiseResult out;
    out.filter_best.h = VectorXd(n);
    out.reconstruction = MatrixXdN(n, problem.channels());
    detail::throw_status(fgfrft_denoise_fit(problem.handle(), e, cfg.lr, cfg.init_alpha, tl.data(), ta.data(),
                                            &out.alpha_best, out.filter_best.h.data(), &out.loss_best,
                                            &out.best_epoch, out.reconstruction.data()));
    out.trajectory.reserve(static_cast<size_t>(e + 1));
    for (int i = 0; i <= e; ++i) out.trajectory.push_back({i, tl[static_cast<size_t>(i)], ta[static_cast<size_t>(i)]});
    return out;
}

}  // namespace fgfrft
