// C++ parity tests of the drop-in header against the reference's own test cases
// (proj/tests/test_transform.cpp, test_sinc.cpp, acceptance.cpp criteria 1-2), compiled against
// include/fgfrft/*.hpp + libfgfrft_b200.so exactly as a reference caller would be.
// Independent checks use tests/oracles.hpp-style mathematics (repeated multiplication,
// closed-form rotations) evaluated on the host, never the library.
// Exit status = number of failed checks.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "fgfrft/fgfrft.hpp"

using namespace fgfrft;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        if (cond) ++g_pass;                                                    \
        else {                                                                 \
            ++g_fail;                                                          \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);        \
        }                                                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                               \
    do {                                                                       \
        bool ok_ = false;                                                      \
        try { (void)(expr); } catch (const T&) { ok_ = true; } catch (...) {}  \
        CHECK(ok_ && #T);                                                      \
    } while (0)

static double max_abs(const MatrixXcd& m) {
    double v = 0;
    for (Index j = 0; j < m.cols(); ++j)
        for (Index i = 0; i < m.rows(); ++i) v = std::max(v, std::abs(m(i, j)));
    return v;
}
static double fro(const MatrixXcd& m) {
    double s = 0;
    for (Index j = 0; j < m.cols(); ++j)
        for (Index i = 0; i < m.rows(); ++i) s += std::norm(m(i, j));
    return std::sqrt(s);
}
static MatrixXcd mul(const MatrixXcd& a, const MatrixXcd& b) {
    MatrixXcd c = MatrixXcd::Zero(a.rows(), b.cols());
    for (Index j = 0; j < b.cols(); ++j)
        for (Index k = 0; k < a.cols(); ++k)
            for (Index i = 0; i < a.rows(); ++i) c(i, j) += a(i, k) * b(k, j);
    return c;
}
static MatrixXcd adj(const MatrixXcd& a) {
    MatrixXcd t(a.cols(), a.rows());
    for (Index j = 0; j < a.cols(); ++j)
        for (Index i = 0; i < a.rows(); ++i) t(j, i) = std::conj(a(i, j));
    return t;
}
static MatrixXcd sub(const MatrixXcd& a, const MatrixXcd& b) {
    MatrixXcd c(a.rows(), a.cols());
    for (Index j = 0; j < a.cols(); ++j)
        for (Index i = 0; i < a.rows(); ++i) c(i, j) = a(i, j) - b(i, j);
    return c;
}
static MatrixXcd eye(Index n) { return MatrixXcd::Identity(n, n); }

// Random unitary as a product of n Householder reflections times a diagonal phase.
static GftMatrix householder_unitary(Index n, unsigned seed) {
    std::mt19937_64 gen(seed);
    std::normal_distribution<double> nd;
    MatrixXcd u = eye(n);
    for (int r = 0; r < 3; ++r) {
        std::vector<std::complex<double>> v(static_cast<size_t>(n));
        double nn = 0;
        for (auto& z : v) { z = {nd(gen), nd(gen)}; nn += std::norm(z); }
        MatrixXcd h = eye(n);
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < n; ++i) h(i, j) -= 2.0 * v[i] * std::conj(v[j]) / nn;
        u = mul(h, u);
    }
    for (Index j = 0; j < n; ++j) {
        const double ph = std::uniform_real_distribution<double>(-M_PI, M_PI)(gen);
        for (Index i = 0; i < n; ++i) u(i, j) *= std::polar(1.0, ph);
    }
    GftMatrix g;
    g.f = u;
    g.provenance = Provenance::haar;
    return g;
}
// Real orthogonal matrix (a product of real Householder reflections): a graph-GFT-like F.
static GftMatrix householder_real(Index n, unsigned seed) {
    std::mt19937_64 gen(seed);
    std::normal_distribution<double> nd;
    MatrixXcd u = eye(n);
    for (int r = 0; r < 4; ++r) {
        std::vector<double> v(static_cast<size_t>(n));
        double nn = 0;
        for (auto& z : v) { z = nd(gen); nn += z * z; }
        MatrixXcd h = eye(n);
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < n; ++i) h(i, j) -= 2.0 * v[i] * v[j] / nn;
        u = mul(h, u);
    }
    GftMatrix g;
    g.f = u;
    g.provenance = Provenance::haar;
    return g;
}
static MatrixXcd matrix_power(const MatrixXcd& f, int m) {  // tests/oracles.hpp:50-56
    MatrixXcd acc = eye(f.rows());
    const MatrixXcd base = m >= 0 ? f : adj(f);
    for (int i = 0; i < std::abs(m); ++i) acc = mul(base, acc);
    return acc;
}
static MatrixXcd rotation2(double phi) {
    MatrixXcd r(2, 2);
    r(0, 0) = std::cos(phi); r(0, 1) = -std::sin(phi);
    r(1, 0) = std::sin(phi); r(1, 1) = std::cos(phi);
    return r;
}

int main() {
    // test_sinc.cpp:9-22, 40-46, 71-73
    {
        const SincCoeffs c0 = sinc_coeffs(0.0, 2);
        for (int n = -2; n <= 2; ++n) CHECK(c0.coeff(n) == (n == 0 ? 1.0 : 0.0));
        const SincCoeffs cm3 = sinc_coeffs(-3.0, 5);
        for (int n = -5; n <= 5; ++n) CHECK(cm3.coeff(n) == (n == -3 ? 1.0 : 0.0));
        for (double a : {0.3, 0.55, 1.0, 1.0000004, 2.5, 1e-8, 7.3}) {
            const SincCoeffs p = sinc_coeffs(a, 6), m = sinc_coeffs(-a, 6);
            for (int n = -6; n <= 6; ++n) CHECK(m.coeff(n) == p.coeff(-n));
        }
        CHECK_THROWS_AS(sinc_coeffs(0.5, 0), parameter_error);
    }
    // test_transform.cpp:20-31
    {
        GftMatrix id;
        id.f = eye(8);
        const PowerCache cache(id, 3);
        for (int k = 1; k <= 3; ++k) CHECK(max_abs(sub(cache.power(k), eye(8))) == 0.0);
        GftMatrix rot;
        rot.f = rotation2(M_PI / 4);
        const PowerCache rc(rot, 4);
        MatrixXcd p4 = rc.power(4);
        for (Index i = 0; i < 2; ++i) p4(i, i) += 1.0;
        CHECK(max_abs(p4) < 1e-14);
    }
    // :33-52 recursion, unitarity, fingerprint, index errors
    {
        const GftMatrix f = householder_unitary(48, 77);
        const PowerCache cache(f, 10);
        CHECK(cache.power(1) == f.f);
        for (int k = 2; k <= 10; ++k) {
            const MatrixXcd step = mul(f.f, cache.power(k - 1));
            CHECK(fro(sub(cache.power(k), step)) <= 1e-9 * fro(step));
        }
        MatrixXcd u = mul(cache.power(10), adj(cache.power(10)));
        for (Index i = 0; i < 48; ++i) u(i, i) -= 1.0;
        CHECK(fro(u) / std::sqrt(48.0) <= 1e-8);
        const GftMatrix other = householder_unitary(48, 78);
        cache.verify(f);
        CHECK_THROWS_AS(cache.verify(other), numerical_error);
        CHECK_THROWS_AS(cache.power(0), parameter_error);
        CHECK_THROWS_AS(cache.power(11), parameter_error);
        CHECK(cache.fingerprint() == content_fingerprint(f.f));
        PowerCache moved = std::move(const_cast<PowerCache&>(cache));
        CHECK(moved.l() == 10 && moved.n() == 48);
        PowerCache copy(moved);
        CHECK(copy.power(7) == moved.power(7));
    }
    // :54-58 memory budget
    {
        const GftMatrix f = householder_unitary(64, 1);
        CHECK_THROWS_AS(PowerCache(f, 10, 1024), capacity_error);
        bool ok = true;
        try { PowerCache(f, 2, 8ull << 20); } catch (...) { ok = false; }
        CHECK(ok);
    }
    // :60-75 order zero exact, integer orders
    {
        const GftMatrix f = householder_unitary(32, 9);
        const PowerCache cache(f, 6);
        CHECK(fro(sub(fgfrft_matrix(cache, 0.0).q, eye(32))) == 0.0);
        const GftMatrix g = householder_unitary(24, 31);
        const PowerCache c2(g, 10);
        for (int m = -3; m <= 3; ++m) {
            const MatrixXcd e = matrix_power(g.f, m);
            CHECK(fro(sub(fgfrft_matrix(c2, double(m)).q, e)) <= 1e-10 * fro(e));
        }
    }
    // :77-85 conjugate symmetry (acceptance criterion 2)
    {
        const PowerCache cache(householder_unitary(40, 13), 10);
        for (double a : {0.3, 0.7, 1.5, 2.2})
            CHECK(max_abs(sub(fgfrft_matrix(cache, -a).q, adj(fgfrft_matrix(cache, a).q))) <= 1e-14);
    }
    // :87-96 quarter rotation: spectral error equals the scalar error (here checked elementwise)
    {
        GftMatrix rot;
        rot.f = rotation2(M_PI / 2);
        const PowerCache cache(rot, 10);
        const MatrixXcd q = fgfrft_matrix(cache, 0.5).q;
        std::complex<double> s = 0;
        for (int n = -10; n <= 10; ++n) s += sinc_coeffs(0.5, 10).coeff(n) * std::polar(1.0, n * M_PI / 2);
        const double scalar_err = std::abs(std::polar(1.0, M_PI / 4) - s);
        CHECK(max_abs(sub(q, rotation2(M_PI / 4))) <= scalar_err + 1e-12);
    }
    // :151-160 gradient vs finite differences
    {
        const PowerCache cache(householder_unitary(32, 15), 10);
        for (double a : {0.15, 0.55, 1.0, 1.5}) {
            MatrixXcd fd = sub(fgfrft_matrix(cache, a + 1e-4).q, fgfrft_matrix(cache, a - 1e-4).q);
            for (Index j = 0; j < 32; ++j)
                for (Index i = 0; i < 32; ++i) fd(i, j) /= 2e-4;
            CHECK(fro(sub(fgfrft_grad(cache, a), fd)) / fro(fd) <= 1e-6);
        }
    }
    // :162-174 identity spectrum gradient
    {
        GftMatrix id;
        id.f = eye(6);
        const PowerCache cache(id, 8);
        CHECK(max_abs(fgfrft_grad(cache, 0.0)) == 0.0);
        const SincCoeffs sc = sinc_coeffs(0.4, 8);
        double sum = 0;
        for (int n = -8; n <= 8; ++n) sum += sc.dcoeff(n);
        const MatrixXcd g = fgfrft_grad(cache, 0.4);
        CHECK(std::abs(g(2, 2).real() - sum) < 1e-14);
        CHECK(std::abs(g(0, 1)) < 1e-14);
    }
    // :176-203 forward / inverse application, shapes
    {
        const GftMatrix f = householder_unitary(64, 40);
        const PowerCache cache(f, 12);
        std::mt19937_64 gen(55);
        std::normal_distribution<double> nd;
        MatrixXcd x(64, 1);
        for (Index i = 0; i < 64; ++i) x(i, 0) = {nd(gen), nd(gen)};
        const FracOperator q0 = fgfrft_matrix(cache, 0.0);
        CHECK(fro(sub(apply_forward(q0, x), x)) == 0.0);
        const FracOperator q1 = fgfrft_matrix(cache, 1.0);
        CHECK(fro(sub(apply_inverse(q1, apply_forward(q1, x)), x)) <= 1e-10 * fro(x));
        const FracOperator q = fgfrft_matrix(cache, 0.7);
        CHECK(fro(sub(apply_series(cache, 0.7, x), mul(q.q, x))) <= 1e-12 * fro(mul(q.q, x)));
        CHECK(fro(sub(apply_series(cache, 0.7, x, true), mul(adj(q.q), x))) <= 1e-12 * fro(x));
        CHECK_THROWS_AS(apply_forward(q, MatrixXcd::Zero(3, 1)), shape_error);
        CHECK_THROWS_AS(apply_inverse(q, MatrixXcd::Zero(3, 1)), shape_error);
        // order gradient: d/da ||Q X - T||^2 via the extension vs finite differences
        MatrixXcd t(64, 1);
        for (Index i = 0; i < 64; ++i) t(i, 0) = {nd(gen), nd(gen)};
        auto loss = [&](double a) { return std::pow(fro(sub(apply_series(cache, a, x), t)), 2); };
        const MatrixXcd r = sub(apply_series(cache, 0.7, x), t);
        MatrixXcd g(64, 1);
        for (Index i = 0; i < 64; ++i) g(i, 0) = 2.0 * r(i, 0);
        const double an = order_gradient(cache, 0.7, g, x);
        const double fd = (loss(0.7 + 1e-5) - loss(0.7 - 1e-5)) / 2e-5;
        CHECK(std::abs(an - fd) <= 1e-6 * std::max(1.0, std::abs(fd)));
    }
    // extension: GEMM engines on a real F (INT8 tensor-core Ozaki engine vs FP64 DMMA)
    {
        const GftMatrix f = householder_real(96, 9);
        PowerCache cache(f, 10);
        cache.prepare();
        std::mt19937_64 gen(56);
        std::normal_distribution<double> nd;
        MatrixXcd x(96, 5);
        for (Index j = 0; j < 5; ++j)
            for (Index i = 0; i < 96; ++i) x(i, j) = {nd(gen), nd(gen)};
        const FracOperator q = fgfrft_matrix(cache, 0.43);
        const MatrixXcd ref = mul(q.q, x);
        cache.set_engine(FGFRFT_ENGINE_INT8);
        const MatrixXcd yi = apply_series(cache, 0.43, x);
        cache.set_engine(FGFRFT_ENGINE_DMMA);
        const MatrixXcd yd = apply_series(cache, 0.43, x);
        CHECK(fro(sub(yi, ref)) <= 1e-11 * fro(ref));
        CHECK(fro(sub(yd, ref)) <= 1e-12 * fro(ref));
        CHECK_THROWS_AS(cache.set_engine(7), parameter_error);
    }
    // :205-221 window warning, truncation override
    {
        const PowerCache cache(householder_unitary(8, 3), 4);
        std::vector<std::string> captured;
        auto previous = warning_sink();
        warning_sink() = [&](const std::string& m) { captured.push_back(m); };
        (void)fgfrft_matrix(cache, 9.0);
        warning_sink() = previous;
        CHECK(!captured.empty() && captured.front().find("window") != std::string::npos);
        CHECK_THROWS_AS(fgfrft_matrix(cache, 0.5, 5), parameter_error);
        CHECK(fgfrft_matrix(cache, 0.5, 2).l == 2);
    }
    // acceptance criterion 1 (N=256, L=10)
    {
        const GftMatrix f = householder_unitary(256, 7);
        const PowerCache cache(f, 10);
        CHECK(fro(sub(fgfrft_matrix(cache, 1.0).q, f.f)) <= 1e-10 * fro(f.f));
        CHECK(fro(sub(fgfrft_matrix(cache, 0.0).q, eye(256))) <= 1e-12 * 16.0);
        const std::vector<MatrixXcd> qs = fgfrft_matrices(cache, {0.0, 1.0});
        CHECK(qs[0] == fgfrft_matrix(cache, 0.0).q && qs[1] == fgfrft_matrix(cache, 1.0).q);
    }
    // spectral.hpp: test_spectral.cpp:34-71, 96-127 through the drop-in header
    {
        const GftMatrix f = householder_unitary(24, 3);
        const UnitaryEigen e = eigendecompose_unitary(f);
        bool ascending = true;
        for (Index k = 1; k < e.theta.size(); ++k) ascending = ascending && e.theta(k - 1) <= e.theta(k);
        CHECK(ascending);
        CHECK(fro(sub(mul(adj(e.v), e.v), eye(24))) <= 1e-12 * std::sqrt(24.0));
        MatrixXcd vd = e.v;
        for (Index j = 0; j < 24; ++j)
            for (Index i = 0; i < 24; ++i) vd(i, j) *= std::polar(1.0, e.theta(j));
        CHECK(fro(sub(mul(f.f, e.v), vd)) <= 1e-9 * fro(f.f));
        CHECK(fro(sub(exact_gfrft(e, 1.0).q, f.f)) <= 1e-12 * fro(f.f));
        CHECK(fro(sub(exact_gfrft(e, 0.0).q, eye(24))) <= 1e-13 * std::sqrt(24.0));
        CHECK(fro(sub(exact_gfrft(e, 2.0).q, mul(f.f, f.f))) <= 1e-12 * fro(f.f));
        const MatrixXcd fd = (exact_gfrft(e, 0.6 + 1e-4).q - exact_gfrft(e, 0.6 - 1e-4).q) * (1.0 / 2e-4);
        CHECK(fro(sub(exact_gfrft_grad(e, 0.6), fd)) <= 1e-6 * fro(fd));
        GftMatrix rot;
        rot.f = MatrixXcd(2, 2);
        const double c = std::cos(M_PI / 4), s = std::sin(M_PI / 4);
        rot.f(0, 0) = c;
        rot.f(0, 1) = -s;
        rot.f(1, 0) = s;
        rot.f(1, 1) = c;
        const UnitaryEigen er = eigendecompose_unitary(rot);
        CHECK(std::fabs(er.theta(0) + M_PI / 4) <= 1e-14 && std::fabs(er.theta(1) - M_PI / 4) <= 1e-14);
        GftMatrix known = f;
        known.known_spectrum = KnownSpectrum{e.v, e.theta};
        const UnitaryEigen ek = eigendecompose_unitary(known);
        CHECK(ek.v == e.v);
        CHECK(fro(sub(exact_gfrft(ek, 0.37).q, exact_gfrft(e, 0.37).q)) <= 1e-13 * std::sqrt(24.0));
        MatrixXcd bad = eye(8);
        bad(0, 1) = 0.5;
        GftMatrix gb;
        gb.f = bad;
        CHECK_THROWS_AS(eigendecompose_unitary(gb), numerical_error);
    }
    // learn.hpp cascade: test_learn.cpp:62-102
    {
        const GftMatrix f = householder_unitary(24, 3);
        for (Backend backend : {Backend::fast, Backend::exact}) {
            for (int k : {1, 3}) {
                CascadeConfig cfg;
                cfg.depth = k;
                cfg.truncation = 8;
                const CascadeProblem problem(f, cfg, backend);
                std::mt19937_64 gen(71 + k);
                std::uniform_real_distribution<double> ud(-0.5, 1.8);
                for (int state = 0; state < 5; ++state) {
                    VectorXd alphas(k);
                    for (int l = 0; l < k; ++l) alphas(l) = ud(gen);
                    const auto ev = problem.eval(alphas);
                    for (int l = 0; l < k; ++l) {
                        VectorXd ap = alphas, am = alphas;
                        ap(l) += 1e-4;
                        am(l) -= 1e-4;
                        const double fdl = (problem.eval(ap).loss - problem.eval(am).loss) / 2e-4;
                        CHECK(std::fabs(ev.grad(l) - fdl) / std::max(std::fabs(fdl), 1e-12) <= 1e-5);
                    }
                }
            }
        }
        CascadeConfig cfg;
        cfg.depth = 1;
        cfg.init_order = 0.7;
        cfg.target_order = 0.7;
        cfg.epochs = 10;
        const OrderLearnResult res = learn_orders(householder_unitary(20, 8), cfg, Backend::exact);
        CHECK(res.final_loss == 0.0);
        CHECK(res.trajectory.size() == 11);
        for (const OrderTrajectoryPoint& p : res.trajectory) CHECK(p.loss == 0.0 && p.alphas[0] == 0.7);
        CascadeConfig c2;
        c2.depth = 2;
        c2.truncation = 30;
        const OrderLearnResult r2 = learn_orders(householder_unitary(48, 21), c2, Backend::fast);
        std::printf("cascade k=2 fast: final loss %.3e, sum(alpha) %.5f\n", r2.final_loss, r2.final_alpha_sum);
        CHECK(std::fabs(r2.final_alpha_sum - 1.5) <= 0.01);
        CHECK(r2.trajectory.back().loss < r2.trajectory.front().loss);
        CascadeConfig bad;
        bad.depth = 0;
        CHECK_THROWS_AS(learn_orders(f, bad, Backend::fast), parameter_error);
    }
    // on-disk cache (extension): save / load round trip, corrupt and missing files
    {
        const GftMatrix f = householder_real(96, 11);
        const PowerCache cache(f, 6);
        const std::string path = "/tmp/fgfrft_dropin_cache.fgc";
        cache.save(path);
        const PowerCache back = PowerCache::load(path);
        CHECK(back.l() == 6 && back.n() == 96 && back.fingerprint() == cache.fingerprint());
        CHECK(back.power(6) == cache.power(6));
        back.verify(f);
        CHECK_THROWS_AS(PowerCache::load("/tmp/fgfrft_no_such_file.fgc"), io_error);
        CHECK_THROWS_AS(PowerCache::load(path, 1024), capacity_error);
        std::remove(path.c_str());
    }
    // learn.hpp denoising: both backends through the drop-in header (acceptance.cpp:183-226 style)
    {
        const GftMatrix f = householder_real(48, 5);
        const Index n = 48;
        std::mt19937_64 gen(600);
        std::normal_distribution<double> nd;
        MatrixXdN x(n, 1), y(n, 1);
        for (Index i = 0; i < n; ++i) {
            x(i, 0) = nd(gen);
            y(i, 0) = x(i, 0) + 0.5 * nd(gen);
        }
        DenoiseConfig cfg;
        cfg.truncation = 8;
        for (Backend backend : {Backend::fast, Backend::exact}) {
            const DenoiseProblem problem(y, x, f, cfg, backend);
            for (int state = 0; state < 3; ++state) {
                const double alpha = -0.5 + 0.9 * state;
                VectorXd h(n);
                for (Index i = 0; i < n; ++i) h(i) = 1.0 + 0.3 * nd(gen);
                const auto ev = problem.eval(alpha, h);
                const double fd = (problem.eval(alpha + 1e-4, h).loss - problem.eval(alpha - 1e-4, h).loss) / 2e-4;
                CHECK(std::fabs(ev.grad_alpha - fd) / std::max(std::fabs(fd), 1e-12) <= 1e-5);
                VectorXd hp = h, hm = h;
                hp(n / 2) += 1e-4;
                hm(n / 2) -= 1e-4;
                const double fdh = (problem.eval(alpha, hp).loss - problem.eval(alpha, hm).loss) / 2e-4;
                CHECK(std::fabs(ev.grad_h(n / 2) - fdh) / std::max(std::fabs(fdh), 1e-12) <= 1e-5);
            }
        }
        cfg.epochs = 20;
        const DenoiseResult r = denoise(y, x, f, cfg, Backend::fast);
        CHECK(r.trajectory.size() == 21);
        CHECK(r.loss_best <= r.trajectory.front().loss);
        CHECK(r.reconstruction.rows() == n && r.reconstruction.cols() == 1);
        const DenoiseResult rc = denoise(y, x, householder_unitary(48, 2), cfg, Backend::fast);  // complex F
        CHECK(rc.trajectory.size() == 21 && rc.loss_best <= rc.trajectory.front().loss);
        DenoiseConfig bad;
        bad.epochs = 0;
        CHECK_THROWS_AS(denoise(y, x, f, bad, Backend::fast), parameter_error);
    }
    std::printf("drop-in C++ tests: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail;
}
