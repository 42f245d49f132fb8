#pragma once
// Graph construction and shift operators (reference: proj/include/fgfrft/graph.hpp). Input
// preparation, not the hot path: with the reference headers on the include path (Eigen builds)
// this forwards to the reference's own header; without Eigen it restates the dense builders the
// reference callers use (grid and k-NN graphs, Laplacian / normalized / adjacency shifts) so that
// they compile unchanged against the drop-in (e.g. demos/fractional_power.cpp).
#include "fgfrft/matrix.hpp"

#if defined(FGFRFT_HAVE_EIGEN) && __has_include_next(<fgfrft/graph.hpp>)
#include_next <fgfrft/graph.hpp>
#else
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>
#include <utility>
#include <vector>

#include "fgfrft/errors.hpp"

namespace fgfrft {

enum class GraphKind { grid, knn, custom };
enum class Normalization { combinatorial_laplacian, symmetric_normalized_laplacian, adjacency };

// Undirected weighted graph as a dense symmetric adjacency (zero diagonal, weights >= 0).
struct Graph {
    Index n = 0;
    MatrixXd adjacency;
    GraphKind kind = GraphKind::custom;

    std::size_t edge_count() const {
        std::size_t e = 0;
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < j; ++i) e += adjacency(i, j) != 0.0;
        return e;
    }
    VectorXd degrees() const {
        VectorXd d(n);
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < n; ++i) d(i) += adjacency(i, j);
        return d;
    }
};

struct ShiftOperator {
    MatrixXd matrix;
    Normalization normalization = Normalization::combinatorial_laplacian;
};

// rows x cols lattice, node (r, c) = r * cols + c, unit edges to the 4 axis neighbours.
inline Graph build_grid_graph(std::int64_t rows, std::int64_t cols) {
    if (rows < 1 || cols < 1) throw parameter_error("build_grid_graph: rows and cols must be >= 1");
    if (rows > std::numeric_limits<std::int32_t>::max() / cols)
        throw capacity_error("build_grid_graph: rows*cols exceeds index range");
    Graph g;
    g.n = static_cast<Index>(rows * cols);
    g.adjacency = MatrixXd::Zero(g.n, g.n);
    g.kind = GraphKind::grid;
    for (std::int64_t r = 0; r < rows; ++r)
        for (std::int64_t c = 0; c < cols; ++c) {
            const Index u = static_cast<Index>(r * cols + c);
            if (c + 1 < cols) g.adjacency(u, u + 1) = g.adjacency(u + 1, u) = 1.0;
            if (r + 1 < rows) g.adjacency(u, u + cols) = g.adjacency(u + cols, u) = 1.0;
        }
    return g;
}

// Symmetrised k-nearest-neighbour graph (unit weights; an edge when either end lists the other).
inline Graph build_knn_graph(const std::vector<std::vector<double>>& points, int k) {
    const Index n = static_cast<Index>(points.size());
    if (n < 2) throw parameter_error("build_knn_graph: need at least two points");
    if (k < 1 || k >= n) throw parameter_error("build_knn_graph: k must be in [1, n)");
    Graph g;
    g.n = n;
    g.adjacency = MatrixXd::Zero(n, n);
    g.kind = GraphKind::knn;
    std::vector<std::pair<double, Index>> d(static_cast<std::size_t>(n));
    for (Index i = 0; i < n; ++i) {
        for (Index j = 0; j < n; ++j) {
            double s = 0.0;
            for (std::size_t t = 0; t < points[i].size(); ++t) {
                const double e = points[i][t] - points[j][t];
                s += e * e;
            }
            d[static_cast<std::size_t>(j)] = {j == i ? std::numeric_limits<double>::infinity() : s, j};
        }
        std::partial_sort(d.begin(), d.begin() + k, d.end());
        for (int q = 0; q < k; ++q) {
            const Index j = d[static_cast<std::size_t>(q)].second;
            g.adjacency(i, j) = g.adjacency(j, i) = 1.0;
        }
    }
    return g;
}

// L = D - A; D^{-1/2} (D - A) D^{-1/2} (isolated nodes give zero rows); or A itself.
inline ShiftOperator shift_operator(const Graph& g, Normalization norm) {
    ShiftOperator z;
    z.normalization = norm;
    z.matrix = MatrixXd::Zero(g.n, g.n);
    const VectorXd deg = g.degrees();
    for (Index j = 0; j < g.n; ++j)
        for (Index i = 0; i < g.n; ++i) {
            const double a = g.adjacency(i, j);
            switch (norm) {
                case Normalization::adjacency: z.matrix(i, j) = a; break;
                case Normalization::combinatorial_laplacian: z.matrix(i, j) = (i == j ? deg(i) : 0.0) - a; break;
                case Normalization::symmetric_normalized_laplacian: {
                    const double si = deg(i) > 0.0 ? 1.0 / std::sqrt(deg(i)) : 0.0;
                    const double sj = deg(j) > 0.0 ? 1.0 / std::sqrt(deg(j)) : 0.0;
                    z.matrix(i, j) = si * ((i == j ? deg(i) : 0.0) - a) * sj;
                    break;
                }
            }
        }
    if (norm == Normalization::symmetric_normalized_laplacian)  // exact symmetry after the scaling
        for (Index j = 0; j < g.n; ++j)
            for (Index i = 0; i < j; ++i) {
                const double m = 0.5 * (z.matrix(i, j) + z.matrix(j, i));
                z.matrix(i, j) = z.matrix(j, i) = m;
            }
    return z;
}

}  // namespace fgfrft
#endif
