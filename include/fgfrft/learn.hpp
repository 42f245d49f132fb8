#pragma once
// Drop-in for the cascaded transform-order learning of proj/include/fgfrft/learn.hpp:25-166,
// backed by libfgfrft_b200.so: the layer operators (series synthesis from the device power cache,
// or the exact spectral form), the prefix products, the reverse gradient accumulation and the
// Adam loop run on the GPU (fgfrft_cascade_*). Same names, fields, error types and messages.
// Divergence: the denoising learner of learn.hpp:168-516 is exposed through the C ABI
// (fgfrft_denoise_*, real F, fast engine) rather than through DenoiseProblem here.

#include <cmath>
#include <cstdint>
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

}  // namespace fgfrft
