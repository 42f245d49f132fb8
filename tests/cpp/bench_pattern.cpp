// The call pattern of the reference's timing_benchmark (proj/include/fgfrft/bench.hpp:150-180) and
// of its acceptance criteria 3 (acceptance.cpp:81-101), compiled against the drop-in include/ as a
// reference caller would be: a synthetic known-spectrum F (gft.hpp synthetic_unitary), its unitary
// eigendecomposition (spectral.hpp), a PowerCache with an explicit budget (transform.hpp:43-59),
// fgfrft_matrix per order and the exact operator for comparison (metrics.hpp matrix_errors).
// Exit status 0 when every check holds.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <vector>

#include "fgfrft/fgfrft.hpp"

int main() {
    using namespace fgfrft;
    int fails = 0;
    for (int n : {96, 160}) {
        Rng rng(Rng::derive(1, static_cast<std::uint64_t>(n)));
        std::vector<double> phases(static_cast<std::size_t>(n));
        for (double& t : phases) t = rng.uniform(-0.95 * M_PI, 0.95 * M_PI);
        const GftMatrix f = synthetic_unitary(phases, 1);
        const UnitaryEigen eig = eigendecompose_unitary(f);
        const PowerCache cache(f, 10, kDefaultMemoryBudget);
        const double alpha = 0.55;
        std::vector<double> t_fast;
        FracOperator fast{};
        for (int r = 0; r < 4; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            fast = fgfrft_matrix(cache, alpha);
            t_fast.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        }
        const FracOperator exact = exact_gfrft(eig, alpha);
        const ErrorReport e = matrix_errors(fast.q, exact.q);
        std::printf("n=%d L=10 alpha=%.2f nmse=%.3e mse=%.3e mae=%.3e fast=%.3es\n", n, alpha, e.nmse, e.mse, e.mae,
                    t_fast.back());
        // L = 10 truncation of a spread spectrum: the paper's regime (NMSE ~ 1e-2, Table II)
        if (!(e.nmse > 1e-5 && e.nmse < 0.2)) ++fails;
        if (unitarity_residual(f.f) > 1e-10) ++fails;
        if (!(phase_margin(f) > 0.0)) ++fails;
    }
    std::printf(fails ? "FAIL %d\n" : "OK\n", fails);
    return fails ? 1 : 0;
}
