#pragma once
// Boundary input type (reference: proj/include/fgfrft/gft.hpp:27-48). F itself is produced by
// the caller's host code (eigendecomposition of the graph shift, Haar sampling, ...).

#include <cstdint>
#include <optional>

#include "fgfrft/matrix.hpp"

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

inline std::uint64_t content_fingerprint(const MatrixXcd& m) {
    return fgfrft_fnv1a64(m.data(), sizeof(std::complex<double>) * static_cast<size_t>(m.rows() * m.cols()));
}

}  // namespace fgfrft
