// Host-only check of the drop-in's no-Eigen input preparation (include/fgfrft/{graph,gft,rng}.hpp):
// prints the grid Laplacian GFT F (gft_from_shift) and a Haar draw (random_unitary) for the Python
// test to compare with prep/ (the numpy restatement of gft.hpp:74-151).
#include <cstdio>

#include "fgfrft/gft.hpp"
#include "fgfrft/graph.hpp"

int main() {
    using namespace fgfrft;
    const GftMatrix f = gft_from_shift(shift_operator(build_grid_graph(5, 6), Normalization::combinatorial_laplacian));
    std::printf("%ld\n", static_cast<long>(f.n()));
    for (Index i = 0; i < f.n(); ++i)
        for (Index j = 0; j < f.n(); ++j) std::printf("%.17g\n", f.f(i, j).real());
    const GftMatrix h = random_unitary(7, 11);
    for (Index i = 0; i < 7; ++i)
        for (Index j = 0; j < 7; ++j) std::printf("%.17g %.17g\n", h.f(i, j).real(), h.f(i, j).imag());
    return 0;
}
