// capi_spectral.cu -- spectral form (eigendecomposition, exact GFRFT) and the cascaded order
// learner (fgfrft_spectrum_*, fgfrft_exact*, fgfrft_cascade_*).
#include "capi_internal.cuh"

// ------------------------------------------------------------------ spectral form, exact GFRFT
//
// spectral.hpp:19-174 on the device: fgfrft_spectrum holds V (n x n,
// complex128, HBM) and the ascending phases theta. The exact operator F^a = V diag(e^{j a theta})
// V^H (and its a-derivative) is one column scaling plus one DMMA complex GEMM per order. The
// decomposition follows eigendecompose_unitary: Hermitian part to cuSOLVER (syevd / heevd), the
// clusters of near-equal cos(theta) rediagonalised against the skew part (small Hermitian
// problems, host Jacobi), Rayleigh quotients, wrap, sort, reconstruction check -- all large
// products on the device.


namespace fgbi {

// cuSOLVER is bound at first use (dlopen), so the library loads without it.
struct SolverApi {
    bool ok = false;
    std::string why;
    decltype(&cusolverDnCreate) create = nullptr;
    decltype(&cusolverDnDestroy) destroy = nullptr;
    decltype(&cusolverDnSetStream) set_stream = nullptr;
    decltype(&cusolverDnDsyevd_bufferSize) dsyevd_bs = nullptr;
    decltype(&cusolverDnDsyevd) dsyevd = nullptr;
    decltype(&cusolverDnZheevd_bufferSize) zheevd_bs = nullptr;
    decltype(&cusolverDnZheevd) zheevd = nullptr;
};

const SolverApi& solver_api() {
    static const SolverApi api = [] {
        SolverApi a;
        void* h = nullptr;
        for (const char* name : {"libcusolver.so.11", "libcusolver.so", "/usr/local/cuda/lib64/libcusolver.so.11"})
            if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) {
            a.why = "cuSOLVER (libcusolver.so.11) is not loadable";
            return a;
        }
        bool all = true;
        auto bind = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            all = all && fp != nullptr;
        };
        bind(a.create, "cusolverDnCreate");
        bind(a.destroy, "cusolverDnDestroy");
        bind(a.set_stream, "cusolverDnSetStream");
        bind(a.dsyevd_bs, "cusolverDnDsyevd_bufferSize");
        bind(a.dsyevd, "cusolverDnDsyevd");
        bind(a.zheevd_bs, "cusolverDnZheevd_bufferSize");
        bind(a.zheevd, "cusolverDnZheevd");
        a.ok = all;
        if (!all) a.why = "cuSOLVER symbols missing";
        return a;
    }();
    return api;
}

using cd = std::complex<double>;

// Eigenpairs of a small Hermitian matrix (column-major k x k, upper triangle used) by cyclic
// complex Jacobi rotations: ascending eigenvalues and orthonormal eigenvectors, the role of the
// cluster SelfAdjointEigenSolver in spectral.hpp:59-64.
void herm_eig_small(int k, std::vector<cd> a, std::vector<cd>& vec) {
    for (int j = 0; j < k; ++j) {
        for (int i = 0; i < j; ++i) a[j + (size_t)i * k] = std::conj(a[i + (size_t)j * k]);
        a[j + (size_t)j * k] = cd(a[j + (size_t)j * k].real(), 0.0);
    }
    vec.assign((size_t)k * k, cd(0.0, 0.0));
    for (int i = 0; i < k; ++i) vec[i + (size_t)i * k] = 1.0;
    double norm2 = 0.0;
    for (const cd& z : a) norm2 += std::norm(z);
    for (int sweep = 0; sweep < 100 && norm2 > 0.0; ++sweep) {
        double off = 0.0;
        for (int q = 0; q < k; ++q)
            for (int p = 0; p < q; ++p) off += std::norm(a[p + (size_t)q * k]);
        if (off <= 1e-32 * norm2) break;
        for (int q = 1; q < k; ++q)
            for (int p = 0; p < q; ++p) {
                const cd apq = a[p + (size_t)q * k];
                const double mag = std::abs(apq);
                if (mag == 0.0) continue;
                const cd ph = std::conj(apq / mag);  // e^{-i phi}
                const double app = a[p + (size_t)p * k].real(), aqq = a[q + (size_t)q * k].real();
                const double tau = (aqq - app) / (2.0 * mag);
                const double t = (tau >= 0.0 ? 1.0 : -1.0) / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
                // J = diag(1, e^{-i phi}) [[c, s], [-s, c]] on (p, q): A <- J^H A J, V <- V J
                const cd jpp = c, jpq = s, jqp = -s * ph, jqq = c * ph;
                for (int r = 0; r < k; ++r) {
                    cd& x = a[r + (size_t)p * k];
                    cd& y = a[r + (size_t)q * k];
                    const cd nx = x * jpp + y * jqp, ny = x * jpq + y * jqq;
                    x = nx;
                    y = ny;
                    cd& vx = vec[r + (size_t)p * k];
                    cd& vy = vec[r + (size_t)q * k];
                    const cd nvx = vx * jpp + vy * jqp, nvy = vx * jpq + vy * jqq;
                    vx = nvx;
                    vy = nvy;
                }
                for (int r = 0; r < k; ++r) {
                    cd& x = a[p + (size_t)r * k];
                    cd& y = a[q + (size_t)r * k];
                    const cd nx = std::conj(jpp) * x + std::conj(jqp) * y, ny = std::conj(jpq) * x + std::conj(jqq) * y;
                    x = nx;
                    y = ny;
                }
                a[p + (size_t)q * k] = a[q + (size_t)p * k] = 0.0;
                a[p + (size_t)p * k] = a[p + (size_t)p * k].real();
                a[q + (size_t)q * k] = a[q + (size_t)q * k].real();
            }
    }
    std::vector<int> ord(k);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(),
                     [&](int x, int y) { return a[x + (size_t)x * k].real() < a[y + (size_t)y * k].real(); });
    std::vector<cd> sorted((size_t)k * k);
    for (int j = 0; j < k; ++j)
        for (int i = 0; i < k; ++i) sorted[i + (size_t)j * k] = vec[i + (size_t)ord[j] * k];
    vec.swap(sorted);
}

struct ScopedBufs {
    DevBuf b[16];
    ~ScopedBufs() {
        for (DevBuf& x : b) x.release();
    }
};

// eigendecompose_unitary (spectral.hpp:121-155) of the host matrix f into s->v / s->theta.
int spectrum_decompose(fgfrft_spectrum* s, const double* f_host) {
    const SolverApi& api = solver_api();
    if (!api.ok) return fail(FGFRFT_NUMERICAL, "eigendecompose_unitary: " + api.why);
    const int n = (int)s->n;
    const size_t nn = (size_t)n * n;
    cudaStream_t st = s->stream;
    bool real = true;  // GftMatrix::is_real, gft.hpp:34-36
    for (size_t i = 0; i < nn && real; ++i) real = std::fabs(f_host[2 * i + 1]) <= 1e-13;
    ScopedBufs sb;
    DevBuf &f = sb.b[0], &a = sb.b[1], &bh = sb.b[2], &w = sb.b[3], &fw = sb.b[4], &t = sb.b[5], &w2 = sb.b[6],
           &fw2 = sb.b[7], &cosv = sb.b[8], &info = sb.b[9], &work = sb.b[10], &pairs = sb.b[11], &vals = sb.b[12],
           &u = sb.b[13], &colinfo = sb.b[14], &part = sb.b[15];
    if (f.ensure(nn * 16) || a.ensure(nn * 16) || bh.ensure(nn * 16) || w.ensure(nn * 16) || fw.ensure(nn * 16) ||
        cosv.ensure((size_t)n * 8) || info.ensure(sizeof(int)) || part.ensure((2 * sp_part_elems() + 2) * 8))
        return fail(FGFRFT_CAPACITY, "eigendecompose_unitary: device allocation failed");
    FGB_CUDA(cudaMemcpyAsync(f.p, f_host, nn * 16, cudaMemcpyHostToDevice, st));
    FGB_LAUNCH(launch_herm_parts(f.p, n, real, a.p, bh.p, st), 1);
    cusolverDnHandle_t h = nullptr;
    if (api.create(&h) != CUSOLVER_STATUS_SUCCESS) return fail(FGFRFT_NUMERICAL, "cusolverDnCreate failed");
    api.set_stream(h, st);
    int lwork = 0;
    cusolverStatus_t cs;
    if (real) {
        cs = api.dsyevd_bs(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, a.as<double>(), n,
                           cosv.as<double>(), &lwork);
        if (cs == CUSOLVER_STATUS_SUCCESS && work.ensure((size_t)std::max(lwork, 1) * 8) == cudaSuccess)
            cs = api.dsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, a.as<double>(), n,
                            cosv.as<double>(), work.as<double>(), lwork, info.as<int>());
    } else {
        cs = api.zheevd_bs(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, a.as<cuDoubleComplex>(), n,
                           cosv.as<double>(), &lwork);
        if (cs == CUSOLVER_STATUS_SUCCESS && work.ensure((size_t)std::max(lwork, 1) * 16) == cudaSuccess)
            cs = api.zheevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, a.as<cuDoubleComplex>(), n,
                            cosv.as<double>(), work.as<cuDoubleComplex>(), lwork, info.as<int>());
    }
    int dev_info = 0;
    const cudaError_t ce = cudaMemcpyAsync(&dev_info, info.p, sizeof(int), cudaMemcpyDeviceToHost, st);
    const cudaError_t se = cudaStreamSynchronize(st);
    api.destroy(h);
    FGB_CUDA(ce);
    FGB_CUDA(se);
    if (cs != CUSOLVER_STATUS_SUCCESS || dev_info != 0)
        return fail(FGFRFT_NUMERICAL, real ? "eigendecompose_unitary: symmetric stage failed"
                                           : "eigendecompose_unitary: Hermitian stage failed");
    if (real)
        FGB_LAUNCH(launch_real_to_cplx(a.as<double>(), (int64_t)nn, w.p, st), 1);
    else
        FGB_CUDA(cudaMemcpyAsync(w.p, a.p, nn * 16, cudaMemcpyDeviceToDevice, st));
    if (int e = zgemm_auto(0, 0, n, n, n, f.p, n, 0, w.p, n, 0, fw.p, n, 0, 1, st)) return e;  // F W
    std::vector<double> cv(n);
    FGB_CUDA(cudaMemcpyAsync(cv.data(), cosv.p, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
    FGB_CUDA(cudaStreamSynchronize(st));
    // clusters of cos(theta) closer than kClusterGap = 1e-5 (spectral.hpp:45, 55-58)
    std::vector<std::pair<int, int>> clusters;  // (lo, k)
    bool any = false;
    for (int lo = 0; lo < n;) {
        int hi = lo;
        while (hi + 1 < n && cv[hi + 1] - cv[hi] <= 1e-5) ++hi;
        clusters.emplace_back(lo, hi - lo + 1);
        any = any || hi > lo;
        lo = hi + 1;
    }
    if (any) {
        // M_c = W_c^H Bh W_c for every cluster of size > 1 (column-major k x k)
        if (t.ensure(nn * 16) || w2.ensure(nn * 16) || fw2.ensure(nn * 16))
            return fail(FGFRFT_CAPACITY, "eigendecompose_unitary: device allocation failed");
        if (int e = zgemm_auto(0, 0, n, n, n, bh.p, n, 0, w.p, n, 0, t.p, n, 0, 1, st)) return e;
        std::vector<int> pr;
        for (const auto& c : clusters)
            if (c.second > 1)
                for (int j = 0; j < c.second; ++j)
                    for (int i = 0; i < c.second; ++i) {
                        pr.push_back(c.first + i);
                        pr.push_back(c.first + j);
                    }
        const int cnt = (int)(pr.size() / 2);
        if (pairs.ensure(pr.size() * sizeof(int)) || vals.ensure((size_t)cnt * 16))
            return fail(FGFRFT_CAPACITY, "eigendecompose_unitary: device allocation failed");
        FGB_CUDA(cudaMemcpyAsync(pairs.p, pr.data(), pr.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        FGB_LAUNCH(launch_col_pair_dot(w.p, t.p, n, pairs.as<int>(), cnt, vals.p, st), 1);
        std::vector<cd> mv((size_t)cnt);
        FGB_CUDA(cudaMemcpyAsync(mv.data(), vals.p, (size_t)cnt * 16, cudaMemcpyDeviceToHost, st));
        FGB_CUDA(cudaStreamSynchronize(st));
        // block-diagonal U: every column gets (lo, k, offset); singletons a 1 x 1 identity block
        std::vector<int> ci((size_t)3 * n);
        std::vector<cd> ub;
        size_t moff = 0;
        for (const auto& c : clusters) {
            const int lo = c.first, k = c.second;
            const int off = (int)ub.size();
            if (k == 1) {
                ub.push_back(1.0);
            } else {
                std::vector<cd> m(mv.begin() + moff, mv.begin() + moff + (size_t)k * k), vec;
                moff += (size_t)k * k;
                herm_eig_small(k, std::move(m), vec);
                ub.insert(ub.end(), vec.begin(), vec.end());
            }
            for (int j = 0; j < k; ++j) {
                ci[3 * (size_t)(lo + j)] = lo;
                ci[3 * (size_t)(lo + j) + 1] = k;
                ci[3 * (size_t)(lo + j) + 2] = off;
            }
        }
        if (u.ensure(ub.size() * 16) || colinfo.ensure(ci.size() * sizeof(int)))
            return fail(FGFRFT_CAPACITY, "eigendecompose_unitary: device allocation failed");
        FGB_CUDA(cudaMemcpyAsync(u.p, ub.data(), ub.size() * 16, cudaMemcpyHostToDevice, st));
        FGB_CUDA(cudaMemcpyAsync(colinfo.p, ci.data(), ci.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        FGB_LAUNCH(launch_blockdiag(w.p, n, colinfo.as<int>(), u.p, w2.p, st), 1);
        FGB_LAUNCH(launch_blockdiag(fw.p, n, colinfo.as<int>(), u.p, fw2.p, st), 1);
        std::swap(w.p, w2.p);
        std::swap(w.cap, w2.cap);
        std::swap(fw.p, fw2.p);
        std::swap(fw.cap, fw2.cap);
        FGB_CUDA(cudaStreamSynchronize(st));  // host staging (ub, ci) is released at scope exit
    }
    // Rayleigh quotients lambda_c = w_c^H F w_c, theta = wrap_phase(lambda) (spectral.hpp:34-38, 67)
    {
        std::vector<int> pr((size_t)2 * n);
        for (int c = 0; c < n; ++c) pr[2 * (size_t)c] = pr[2 * (size_t)c + 1] = c;
        if (pairs.ensure(pr.size() * sizeof(int)) || vals.ensure((size_t)n * 16))
            return fail(FGFRFT_CAPACITY, "eigendecompose_unitary: device allocation failed");
        FGB_CUDA(cudaMemcpyAsync(pairs.p, pr.data(), pr.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        FGB_LAUNCH(launch_col_pair_dot(w.p, fw.p, n, pairs.as<int>(), n, vals.p, st), 1);
        std::vector<cd> lam((size_t)n);
        FGB_CUDA(cudaMemcpyAsync(lam.data(), vals.p, (size_t)n * 16, cudaMemcpyDeviceToHost, st));
        FGB_CUDA(cudaStreamSynchronize(st));
        std::vector<double> th((size_t)n);
        for (int c = 0; c < n; ++c) {
            double tv = std::atan2(lam[c].imag(), lam[c].real());
            if (tv <= -M_PI) tv = M_PI;
            th[c] = tv;
        }
        // reconstruction residual |F W - W diag(e^{j theta})| / |F| <= 1e-6 (spectral.hpp:141-153)
        FGB_CUDA(cudaMemcpyAsync(cosv.p, th.data(), (size_t)n * 8, cudaMemcpyHostToDevice, st));
        double* pp = part.as<double>();
        FGB_CUDA(launch_eig_residual(fw.p, w.p, cosv.as<double>(), f.p, n, pp, pp + 2 * sp_part_elems(), st));
        g_launches += 2;
        double rr[2] = {0.0, 0.0};
        FGB_CUDA(cudaMemcpyAsync(rr, pp + 2 * sp_part_elems(), 16, cudaMemcpyDeviceToHost, st));
        FGB_CUDA(cudaStreamSynchronize(st));
        const double rel = std::sqrt(rr[0]) / std::max(std::sqrt(rr[1]), 1e-300);
        if (!(rel <= 1e-6)) {
            std::ostringstream msg;
            msg << "eigendecompose_unitary: reconstruction residual " << rel << " exceeds 1e-6";
            return fail(FGFRFT_NUMERICAL, msg.str());
        }
        std::vector<int> order((size_t)n);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return th[x] < th[y]; });
        s->theta_h.resize((size_t)n);
        for (int c = 0; c < n; ++c) s->theta_h[c] = th[order[c]];
        if (s->v.ensure(nn * 16) || s->theta.ensure((size_t)n * 8))
            return fail(FGFRFT_CAPACITY, "eigendecompose_unitary: device allocation failed");
        FGB_CUDA(cudaMemcpyAsync(pairs.p, order.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice, st));
        FGB_LAUNCH(launch_gather_cols(w.p, n, pairs.as<int>(), s->v.p, st), 1);
        FGB_CUDA(cudaMemcpyAsync(s->theta.p, s->theta_h.data(), (size_t)n * 8, cudaMemcpyHostToDevice, st));
        FGB_CUDA(cudaStreamSynchronize(st));
    }
    return FGFRFT_OK;
}

// out[a] = V diag(d_a) V^H for the orders (which: FGFRFT_Q or FGFRFT_DQ), spectral.hpp:158-174.
int exact_into(fgfrft_spectrum* s, const double* alphas, int na, int which, void* out, cudaStream_t st) {
    const int n = (int)s->n;
    const size_t nn = (size_t)n * n;
    const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)na, ((size_t)2 << 30) / (nn * 16)));
    FGB_CUDA(s->alph.ensure((size_t)na * 8));
    FGB_CUDA(s->w.ensure((size_t)chunk * nn * 16));
    FGB_CUDA(cudaMemcpyAsync(s->alph.p, alphas, (size_t)na * 8, cudaMemcpyHostToDevice, st));
    for (int a0 = 0; a0 < na; a0 += chunk) {
        const int nc = std::min(chunk, na - a0);
        FGB_LAUNCH(launch_spec_scale(s->v.p, s->theta.as<double>(), s->alph.as<double>() + a0, nc, which, n, s->w.p,
                                     st),
                   1);
        if (int e = zgemm_auto(0, 2, n, n, n, s->w.p, n, (int64_t)nn, s->v.p, n, 0,
                               static_cast<double2*>(out) + (size_t)a0 * nn, n, (int64_t)nn, nc, st))
            return e;
    }
    return FGFRFT_OK;
}

int check_spectrum(const fgfrft_spectrum* s) {
    if (!s) return fail(FGFRFT_PARAMETER, "null fgfrft_spectrum handle");
    return FGFRFT_OK;
}

int spectrum_new(int64_t n, int device, fgfrft_spectrum** out) {
    auto* s = new fgfrft_spectrum();
    s->n = n;
    s->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete s;
        return fail(FGFRFT_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    s->stream = s->own_stream;
    *out = s;
    return FGFRFT_OK;
}

void spectrum_free(fgfrft_spectrum* s) {
    if (s->stream) cudaStreamSynchronize(s->stream);
    for (DevBuf* b : {&s->v, &s->theta, &s->alph, &s->w}) b->release();
    if (s->own_stream) cudaStreamDestroy(s->own_stream);
    delete s;
}

// ---- cascade (learn.hpp:55-166)

// loss and per-layer gradients at the host orders: out_host[0] = loss, out_host[1 + l] = grad_l.
//   forward: prefix_l = Q_l prefix_{l-1}, resid = prefix_{K-1} - target, loss = |resid|^2 / N^2
//   reverse: grad_l = 2/N^2 Re<b, dQ_l prefix_{l-1}>, b <- Q_l^H b           (learn.hpp:72-97)
// Complex F: Re<b, dQ X> is taken as Re<b X^H, dQ> (complex GEMMs on the FP64 tensor cores).
// Real F (fast backend): Q_l, dQ_l and the prefixes are real, so the products are real DMMA GEMMs
// (dQ_l prefix_{l-1} real x real, Q_l^T b real x complex): a third of the complex flops.
int cascade_eval_device(fgfrft_cascade* cs, const double* alphas, double* out_host) {
    const int K = cs->k;
    const int n = (int)cs->n;
    const size_t nn = (size_t)n * n;
    cudaStream_t st = cs->stream();
    const bool real = cs->cache && cs->cache->real;
    const size_t es = real ? 8 : 16;
    char* ops = cs->ops.as<char>();
    char* dops = cs->dops.as<char>();
    if (cs->cache) {
        fgfrft_cache* c = cs->cache;
        double* coef = nullptr;
        if (int e = upload_coefs(c, alphas, K, c->l, &coef)) return e;
        if (int e = synth_into(c, coef, K, c->l, ops, real)) return e;
        if (int e = synth_into(c, coef + (size_t)K * (2 * c->l + 1), K, c->l, dops, real)) return e;
    } else {
        if (int e = exact_into(cs->spec, alphas, K, FGFRFT_Q, ops, st)) return e;
        if (int e = exact_into(cs->spec, alphas, K, FGFRFT_DQ, dops, st)) return e;
    }
    auto op = [&](char* base, int l) { return static_cast<void*>(base + (size_t)l * nn * es); };
    auto prefix = [&](int l) { return l == 0 ? op(ops, 0) : op(cs->prefix.as<char>(), l); };
    // real x real products: INT8 Ozaki engine where the cache's engine selects it, else DMMA
    const bool i8 = real && use_int8_gemm(cs->cache, n);
    auto real_mm = [&](const void* a, const void* bb, void* cc) -> int {
        if (i8)
            return fgfrft_dgemm_int8_dev(0, 0, n, n, n, static_cast<const double*>(a), n,
                                         static_cast<const double*>(bb), n, static_cast<double*>(cc), n, 0, st);
        ProfScope ps(KC_GEMM, st);
        FGB_LAUNCH(launch_rgemm(0, 0, 0, n, n, n, a, n, 0, bb, n, 0, cc, n, 0, 1, st), 1);
        return FGFRFT_OK;
    };
    for (int l = 1; l < K; ++l) {
        if (real) {
            if (int e = real_mm(op(ops, l), prefix(l - 1), prefix(l))) return e;
            continue;
        }
        if (int e = zgemm_auto(0, 0, n, n, n, op(ops, l), n, 0, prefix(l - 1), n, 0, prefix(l), n, 0, 1, st)) return e;
    }
    double* part = cs->part.as<double>();
    const size_t G = sp_part_elems();
    double2* b = cs->b.as<double2>();
    double2* nb = cs->nb.as<double2>();
    FGB_LAUNCH(launch_cdiff_sq(prefix(K - 1), real, cs->target.p, (int64_t)nn, b, part, st), 1);
    for (int l = K - 1; l >= 0; --l) {
        if (l > 0) {
            {
                ProfScope ps(KC_GEMM, st);
                if (real) {  // dY = dQ_l prefix_{l-1}
                    if (int e = real_mm(op(dops, l), prefix(l - 1), cs->m.p)) return e;
                } else {  // M = b prefix_{l-1}^H
                    if (int e = zgemm_auto(0, 2, n, n, n, b, n, 0, prefix(l - 1), n, 0, cs->m.p, n, 0, 1, st))
                        return e;
                }
            }
            if (real)
                FGB_LAUNCH(launch_cre_dot(b, cs->m.p, true, (int64_t)nn, part + (1 + l) * G, st), 1);
            else
                FGB_LAUNCH(launch_cre_dot(cs->m.p, op(dops, l), false, (int64_t)nn, part + (1 + l) * G, st), 1);
            ProfScope ps(KC_GEMM, st);
            if (i8) {  // b <- Q_l^T b
                if (int e = int8_qx(cs->cache, 1, true, op(ops, l), b, n, nb)) return e;
            } else if (real) {  // over the (re, im) columns
                FGB_LAUNCH(launch_rgemm(1, 1, 1, n, 2 * n, n, op(ops, l), n, 0, b, n, 0, nb, n, 0, 1, st), 1);
            } else if (int e = zgemm_auto(2, 0, n, n, n, op(ops, l), n, 0, b, n, 0, nb, n, 0, 1, st)) {
                return e;
            }
            std::swap(b, nb);
        } else {
            FGB_LAUNCH(launch_cre_dot(b, dops, real, (int64_t)nn, part + G, st), 1);
        }
    }
    const double inv = 1.0 / ((double)n * (double)n);
    FGB_LAUNCH(launch_sum_parts(part, K + 1, inv, 2.0 * inv, cs->out.as<double>(), st), 1);
    FGB_CUDA(cudaMemcpyAsync(out_host, cs->out.p, (size_t)(K + 1) * 8, cudaMemcpyDeviceToHost, st));
    FGB_CUDA(cudaStreamSynchronize(st));
    return FGFRFT_OK;
}

int check_cascade(const fgfrft_cascade* cs) {
    if (!cs || !cs->spec) return fail(FGFRFT_PARAMETER, "null fgfrft_cascade handle");
    return FGFRFT_OK;
}

// Locks the handle(s) the cascade computes through.
struct CascadeLock {
    std::unique_lock<std::mutex> a, b;
    explicit CascadeLock(fgfrft_cascade* cs) : b(cs->spec->mu) {
        if (cs->cache) a = std::unique_lock<std::mutex>(cs->cache->mu);
    }
};

}  // namespace fgbi

extern "C" {

int fgfrft_spectrum_create(const double* v, const double* theta, int64_t n, int device, fgfrft_spectrum** out) {
    FGB_GUARD_BEGIN
    if (!out) return fail(FGFRFT_PARAMETER, "null output handle pointer");
    *out = nullptr;
    if (n < 1) return fail(FGFRFT_SHAPE, "spectrum: n must be >= 1");
    if (!v || !theta) return fail(FGFRFT_PARAMETER, "null spectrum buffer");
    for (int64_t k = 0; k < n; ++k)
        if (!std::isfinite(theta[k])) return fail(FGFRFT_PARAMETER, "spectrum: phases must be finite");
    DeviceGuard dg(device);
    fgfrft_spectrum* s = nullptr;
    if (int st = spectrum_new(n, device, &s)) return st;
    const size_t nn = (size_t)n * n;
    int rc = FGFRFT_OK;
    if (s->v.ensure(nn * 16) || s->theta.ensure((size_t)n * 8))
        rc = fail(FGFRFT_CAPACITY, "spectrum: device allocation failed");
    if (rc == FGFRFT_OK) {
        s->theta_h.assign(theta, theta + n);
        if (cudaMemcpyAsync(s->v.p, v, nn * 16, cudaMemcpyHostToDevice, s->stream) ||
            cudaMemcpyAsync(s->theta.p, theta, (size_t)n * 8, cudaMemcpyHostToDevice, s->stream) ||
            cudaStreamSynchronize(s->stream))
            rc = fail(FGFRFT_CUDA, "spectrum: upload failed");
    }
    if (rc != FGFRFT_OK) {
        spectrum_free(s);
        return rc;
    }
    *out = s;
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_spectrum_decompose(const double* f, int64_t n, int device, fgfrft_spectrum** out) {
    FGB_GUARD_BEGIN
    if (!out) return fail(FGFRFT_PARAMETER, "null output handle pointer");
    *out = nullptr;
    if (n < 1) return fail(FGFRFT_SHAPE, "eigendecompose_unitary: n must be >= 1");
    if (n > (1 << 15)) return fail(FGFRFT_SHAPE, "eigendecompose_unitary: n too large");
    if (!f) return fail(FGFRFT_PARAMETER, "null matrix");
    DeviceGuard dg(device);
    fgfrft_spectrum* s = nullptr;
    if (int st = spectrum_new(n, device, &s)) return st;
    if (int st = spectrum_decompose(s, f)) {
        spectrum_free(s);
        return st;
    }
    *out = s;
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_spectrum_destroy(fgfrft_spectrum* s) {
    if (!s) return FGFRFT_OK;
    DeviceGuard dg(s->device);
    spectrum_free(s);
    return FGFRFT_OK;
}

int fgfrft_spectrum_info(const fgfrft_spectrum* s, int64_t* n, double* theta) {
    if (int st = check_spectrum(s)) return st;
    if (n) *n = s->n;
    if (theta) std::memcpy(theta, s->theta_h.data(), (size_t)s->n * 8);
    return FGFRFT_OK;
}

int fgfrft_spectrum_vectors(fgfrft_spectrum* s, double* v) {
    FGB_GUARD_BEGIN
    if (int st = check_spectrum(s)) return st;
    if (!v) return fail(FGFRFT_PARAMETER, "null output");
    std::lock_guard<std::mutex> lk(s->mu);
    DeviceGuard dg(s->device);
    FGB_CUDA(cudaMemcpyAsync(v, s->v.p, (size_t)s->n * s->n * 16, cudaMemcpyDeviceToHost, s->stream));
    FGB_CUDA(cudaStreamSynchronize(s->stream));
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_spectrum_set_stream(fgfrft_spectrum* s, void* stream) {
    if (int st = check_spectrum(s)) return st;
    std::lock_guard<std::mutex> lk(s->mu);
    s->stream = stream ? static_cast<cudaStream_t>(stream) : s->own_stream;
    return FGFRFT_OK;
}

int fgfrft_exact_dev(fgfrft_spectrum* s, const double* alphas, int n_alpha, int which, void* out_dev) {
    FGB_GUARD_BEGIN
    if (int st = check_spectrum(s)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (which != FGFRFT_Q && which != FGFRFT_DQ) return fail(FGFRFT_PARAMETER, "which must be FGFRFT_Q or FGFRFT_DQ");
    if (!out_dev) return fail(FGFRFT_PARAMETER, "null output");
    std::lock_guard<std::mutex> lk(s->mu);
    DeviceGuard dg(s->device);
    return exact_into(s, alphas, n_alpha, which, out_dev, s->stream);
    FGB_GUARD_END
}

int fgfrft_exact(fgfrft_spectrum* s, const double* alphas, int n_alpha, int which, double* out) {
    FGB_GUARD_BEGIN
    if (int st = check_spectrum(s)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (which != FGFRFT_Q && which != FGFRFT_DQ) return fail(FGFRFT_PARAMETER, "which must be FGFRFT_Q or FGFRFT_DQ");
    if (!out) return fail(FGFRFT_PARAMETER, "null output");
    std::lock_guard<std::mutex> lk(s->mu);
    DeviceGuard dg(s->device);
    const size_t nn = (size_t)s->n * s->n;
    DevBuf o;
    if (o.ensure((size_t)n_alpha * nn * 16)) return fail(FGFRFT_CAPACITY, "exact_gfrft: device allocation failed");
    int rc = exact_into(s, alphas, n_alpha, which, o.p, s->stream);
    if (rc == FGFRFT_OK &&
        (cudaMemcpyAsync(out, o.p, (size_t)n_alpha * nn * 16, cudaMemcpyDeviceToHost, s->stream) ||
         cudaStreamSynchronize(s->stream)))
        rc = fail(FGFRFT_CUDA, "exact_gfrft: download failed");
    o.release();
    return rc;
    FGB_GUARD_END
}

int fgfrft_cascade_create(fgfrft_cache* cache, fgfrft_spectrum* spec, double target_order, int depth,
                          fgfrft_cascade** out) {
    FGB_GUARD_BEGIN
    if (!out) return fail(FGFRFT_PARAMETER, "null output handle pointer");
    *out = nullptr;
    if (int st = check_spectrum(spec)) return st;
    if (depth < 1) return fail(FGFRFT_PARAMETER, "CascadeConfig: depth must be >= 1");
    if (!std::isfinite(target_order)) return fail(FGFRFT_PARAMETER, "CascadeConfig: target order must be finite");
    if (cache) {
        if (int st = check_handle(cache)) return st;
        if (cache->dtype != FGFRFT_C128) return fail(FGFRFT_PARAMETER, "cascade: the fast backend needs a complex128 cache");
        if (cache->n != spec->n) return fail(FGFRFT_SHAPE, "cascade: cache and spectrum sizes differ");
        if (cache->device != spec->device) return fail(FGFRFT_PARAMETER, "cascade: cache and spectrum on different devices");
    }
    std::lock_guard<std::mutex> lk(spec->mu);
    DeviceGuard dg(spec->device);
    auto* cs = new fgfrft_cascade();
    cs->cache = cache;
    cs->spec = spec;
    cs->k = depth;
    cs->n = spec->n;
    const size_t blk = (size_t)cs->n * cs->n * 16;
    int rc = FGFRFT_OK;
    if (cs->target.ensure(blk) || cs->ops.ensure((size_t)depth * blk) || cs->dops.ensure((size_t)depth * blk) ||
        cs->prefix.ensure((size_t)depth * blk) || cs->b.ensure(blk) || cs->nb.ensure(blk) ||
        (depth > 1 && cs->m.ensure(blk)) || cs->part.ensure((size_t)(depth + 1) * sp_part_elems() * 8) ||
        cs->out.ensure((size_t)(depth + 1) * 8))
        rc = fail(FGFRFT_CAPACITY, "cascade: device allocation failed");
    // target = F^{target_order} from the spectrum, always exact (learn.hpp:61)
    if (rc == FGFRFT_OK) rc = exact_into(spec, &target_order, 1, FGFRFT_Q, cs->target.p, spec->stream);
    if (rc == FGFRFT_OK && cudaStreamSynchronize(spec->stream) != cudaSuccess)
        rc = fail(FGFRFT_CUDA, "cascade: target construction failed");
    if (rc != FGFRFT_OK) {
        for (DevBuf* b : {&cs->target, &cs->ops, &cs->dops, &cs->prefix, &cs->b, &cs->nb, &cs->m, &cs->part, &cs->out})
            b->release();
        delete cs;
        return rc;
    }
    *out = cs;
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_cascade_destroy(fgfrft_cascade* cs) {
    if (!cs) return FGFRFT_OK;
    if (cs->spec) {
        DeviceGuard dg(cs->spec->device);
        cudaStreamSynchronize(cs->stream());
    }
    for (DevBuf* b : {&cs->target, &cs->ops, &cs->dops, &cs->prefix, &cs->b, &cs->nb, &cs->m, &cs->part, &cs->out})
        b->release();
    delete cs;
    return FGFRFT_OK;
}

int fgfrft_cascade_eval(fgfrft_cascade* cs, const double* alphas, double* loss, double* grad) {
    FGB_GUARD_BEGIN
    if (int st = check_cascade(cs)) return st;
    if (!alphas) return fail(FGFRFT_PARAMETER, "null orders");
    if (int st = check_alphas(alphas, cs->k)) return st;
    CascadeLock lk(cs);
    DeviceGuard dg(cs->spec->device);
    std::vector<double> o((size_t)cs->k + 1);
    if (int st = cascade_eval_device(cs, alphas, o.data())) return st;
    if (loss) *loss = o[0];
    if (grad) std::memcpy(grad, o.data() + 1, (size_t)cs->k * 8);
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_cascade_learn(fgfrft_cascade* cs, double init_order, int epochs, double lr, double* traj_loss,
                         double* traj_alphas, double* final_loss, double* final_alphas) {
    FGB_GUARD_BEGIN
    if (int st = check_cascade(cs)) return st;
    if (epochs < 1) return fail(FGFRFT_PARAMETER, "CascadeConfig: epochs must be >= 1");
    if (!(lr > 0.0)) return fail(FGFRFT_PARAMETER, "CascadeConfig: lr must be positive");
    if (!std::isfinite(init_order)) return fail(FGFRFT_PARAMETER, "CascadeConfig: init order must be finite");
    CascadeLock lk(cs);
    DeviceGuard dg(cs->spec->device);
    const int K = cs->k;
    // AdamState::init(constant(init_order), lr), adam_step (adam.hpp:24-53)
    std::vector<double> p((size_t)K, init_order), m((size_t)K, 0.0), v((size_t)K, 0.0), o((size_t)K + 1);
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    int64_t step = 0;
    auto record = [&](int e, double l) {
        if (traj_loss) traj_loss[e] = l;
        if (traj_alphas) std::memcpy(traj_alphas + (size_t)e * K, p.data(), (size_t)K * 8);
    };
    for (int e = 0; e < epochs; ++e) {  // learn.hpp:142-152
        if (int st = cascade_eval_device(cs, p.data(), o.data())) return st;
        if (!std::isfinite(o[0])) {
            std::ostringstream msg;
            msg << "learn_orders: non-finite loss at epoch " << e;
            return fail(FGFRFT_OPTIMIZER, msg.str());
        }
        record(e, o[0]);
        for (int i = 0; i < K; ++i)
            if (!std::isfinite(o[1 + i])) {
                std::ostringstream msg;
                msg << "adam_step: non-finite gradient at step " << step + 1 << ", parameter " << i;
                return fail(FGFRFT_OPTIMIZER, msg.str());
            }
        ++step;
        const double c1 = 1.0 - std::pow(b1, (double)step), c2 = 1.0 - std::pow(b2, (double)step);
        for (int i = 0; i < K; ++i) {
            const double g = o[1 + i];
            m[i] = b1 * m[i] + (1.0 - b1) * g;
            v[i] = b2 * v[i] + (1.0 - b2) * (g * g);
            p[i] = p[i] - lr * (m[i] / c1) / (std::sqrt(v[i] / c2) + eps);
        }
    }
    if (int st = cascade_eval_device(cs, p.data(), o.data())) return st;  // learn.hpp:154-155
    record(epochs, o[0]);
    if (final_loss) *final_loss = o[0];
    if (final_alphas) std::memcpy(final_alphas, p.data(), (size_t)K * 8);
    return FGFRFT_OK;
    FGB_GUARD_END
}

}  // extern "C"
