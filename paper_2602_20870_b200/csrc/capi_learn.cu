// capi_learn.cu -- the GPU-resident denoising learner: fast (synthesised Q, dQ from the power
// cache) and exact (device spectrum) backends, Adam on the device (fgfrft_denoise_*).
#include "capi_internal.cuh"

// ------------------------------------------------------------------ GPU-resident denoising learner
//
// learn.hpp:291-413 (FastDenoiseEngine, real F) and learn.hpp:471-516 (denoise + Adam, adam.hpp)
// on the device. Kernels: denoise.cu (pieces), the pair synthesis (Q and dQ/dalpha from the
// cache), the INT8 / DMMA real GEMMs.


namespace fgbi {

// handle plumbing shared by both backends (defined after fgfrft_spectrum)
cudaStream_t dn_stream(const fgfrft_denoise* d);
std::mutex& dn_mutex(fgfrft_denoise* d);
int dn_device(const fgfrft_denoise* d);
int denoise_exact_eval(fgfrft_denoise* d, const double* params, double* loss, double* grad, int epoch);

// C (n x ch) = op(A) B for real n x n A (op: A or A^T) and real n x ch B, column-major: the INT8
// engine where the cache's engine selects it, else a real DMMA GEMM.
int dn_gemm(fgfrft_cache* c, bool trans, const double* a, const double* b, double* out, int64_t ch) {
    const int64_t n = c->n;
    if (use_int8_gemm(c, (ch + 1) / 2))
        return fgfrft_dgemm_int8_dev(trans ? 1 : 0, 0, n, ch, n, a, n, b, n, out, n, 0, c->stream);
    ProfScope ps(KC_GEMM, c->stream);
    FGB_LAUNCH(launch_rgemm(trans ? 1 : 0, 0, 0, (int)n, (int)ch, (int)n, a, n, 0, b, n, 0, out, n, 0, 1, c->stream),
               1);
    return FGFRFT_OK;
}

// One evaluation at the device-resident params = [alpha, h_1..h_n]: loss, grad = [d/dalpha, d/dh].
// The reference's matrix-free engine (learn.hpp:291-413) applies Q = sum_m c_m F^m through 4L
// products with F per evaluation; here Q and dQ/dalpha are synthesised together from the device
// cache (one pass, the pair kernel's 2-order form: exact, P_-m = P_m^T) and every "sum_m c_m F^m
// applied to a block" becomes one GEMM:
//   u = Q y, du = dQ y, v = h o u, w = Q^T v (= sum c_-m F^m v), dqh_v = dQ^T v, r = w - x,
//   qr = Q r, grad_h = 2 rowsum(qr o u), grad_alpha = 2 <r, dqh_v> + 2 <qr, h o du>.
// Complex F (FastDenoiseEngine<MatrixXcd>): the same five products as complex GEMMs (INT8 engine
// from n = 512, else DMMA), Q^H / dQ^H as conjugate-transposed operands; the scalings and
// reductions are the exact backend's kernels (dnx_*; the "jtc" diagonal is all ones here).
int denoise_fast_complex_eval(fgfrft_denoise* d, const double* params, double* loss, double* grad, int epoch) {
    fgfrft_cache* c = d->cache;
    cudaStream_t st = c->stream;
    const int n = (int)d->n, ch = (int)d->ch;
    const int64_t cnt = (int64_t)n * ch;
    const size_t nn = (size_t)n * n;
    const double* h = params + 1;
    double* tab = d->tab.as<double>();
    double2* q = d->qd.as<double2>();
    double2* dq = q + nn;
    auto zg = [&](int opa, const void* a, const void* b, void* out) {
        return zgemm_auto(opa, 0, n, ch, n, a, n, 0, b, n, 0, out, n, 0, 1, st);
    };
    FGB_LAUNCH(launch_dn_coef(params, d->l, tab, st), 1);
    if (int e = synth_into(c, tab, 2, d->l, q, true)) return e;
    if (int e = zg(0, q, d->xytil.p, d->xu.p)) return e;                  // u = Q y
    if (int e = zg(0, dq, d->xytil.p, d->xb.p)) return e;                 // du = dQ y
    FGB_LAUNCH(launch_dnx_rowscale(d->xu.p, nullptr, h, false, n, cnt, d->xq.p, st), 1);  // v = h o u
    if (int e = zg(2, q, d->xq.p, d->xw.p)) return e;                     // w = Q^H v
    if (int e = zg(2, dq, d->xq.p, d->xvhr.p)) return e;                  // dQ^H v
    double* part = d->part.as<double>();
    FGB_LAUNCH(launch_dnx_cot(d->xw.p, d->x.as<double>(), cnt, d->loss_on_real, d->xcot.p, part, st), 1);
    if (int e = zg(0, q, d->xcot.p, d->xfar.p)) return e;                 // qr = Q r
    FGB_LAUNCH(launch_dnx_grad(d->xfar.p, d->xu.p, d->xcot.p, d->xvhr.p, d->xph.p, d->xb.p, h, n, ch, grad + 1, part,
                               st),
               1);
    FGB_LAUNCH(launch_dn_finish(part, loss, grad, n, d->flag.as<int>(), epoch, st), 1);
    return FGFRFT_OK;
}

int denoise_eval_device(fgfrft_denoise* d, const double* params, double* loss, double* grad, int epoch = -1) {
    if (d->exact) return denoise_exact_eval(d, params, loss, grad, epoch);
    if (d->cplx) return denoise_fast_complex_eval(d, params, loss, grad, epoch);
    fgfrft_cache* c = d->cache;
    const int l = d->l;
    const int64_t cnt = d->n * d->ch, cp = d->cpad, ch = d->ch;
    const size_t nn = (size_t)d->n * d->n;
    double* tab = d->tab.as<double>();
    const double* h = params + 1;
    double* q = d->qd.as<double>();
    double* dq = q + nn;
    double* uu = d->uu.as<double>();
    double* ww = d->ww.as<double>();
    FGB_LAUNCH(launch_dn_coef(params, l, tab, c->stream), 1);  // rows c(alpha), c'(alpha)
    if (int st = synth_into(c, tab, 2, l, q, true)) return st;
    if (int st = dn_gemm(c, false, q, d->y.as<double>(), uu, ch)) return st;        // u
    if (int st = dn_gemm(c, false, dq, d->y.as<double>(), uu + cp, ch)) return st;  // du
    FGB_LAUNCH(launch_dn_scale(uu, h, d->v.as<double>(), (int)d->n, cnt, c->stream), 1);
    if (int st = dn_gemm(c, true, q, d->v.as<double>(), ww, ch)) return st;         // w = Q^T v
    if (int st = dn_gemm(c, true, dq, d->v.as<double>(), ww + cp, ch)) return st;   // dQ^T v
    double* part = d->part.as<double>();
    FGB_LAUNCH(launch_dn_residual(ww, d->x.as<double>(), d->r.as<double>(), cnt, part, c->stream), 1);
    if (int st = dn_gemm(c, false, q, d->r.as<double>(), d->qr.as<double>(), ch)) return st;  // qr = Q r
    FGB_LAUNCH(launch_dn_grad(uu, uu + cp, h, d->r.as<double>(), ww + cp, d->qr.as<double>(), (int)d->n, (int)d->ch,
                              grad, part, loss, d->flag.as<int>(), epoch, c->stream),
               2);
    return FGFRFT_OK;
}

int check_denoise(const fgfrft_denoise* d) {
    if (!d || (!d->cache && !d->spec)) return fail(FGFRFT_PARAMETER, "null fgfrft_denoise handle");
    return FGFRFT_OK;
}

}  // namespace fgbi

extern "C" {

int fgfrft_denoise_create(fgfrft_cache* c, const double* y, const double* x_ref, int64_t channels,
                          fgfrft_denoise** out) {
    return fgfrft_denoise_create_ex(c, y, x_ref, channels, 0, out);
}

int fgfrft_denoise_create_ex(fgfrft_cache* c, const double* y, const double* x_ref, int64_t channels,
                             int loss_on_real, fgfrft_denoise** out) {
    FGB_GUARD_BEGIN
    if (!out) return fail(FGFRFT_PARAMETER, "null output handle pointer");
    *out = nullptr;
    if (int st = check_handle(c)) return st;
    if (c->dtype != FGFRFT_C128 || c->api_c64)
        return fail(FGFRFT_PARAMETER, "denoise on the device needs a complex128 cache");
    if (channels < 1) return fail(FGFRFT_SHAPE, "denoise: need at least one channel");
    if (!y || !x_ref) return fail(FGFRFT_PARAMETER, "null signal buffer");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    auto* d = new fgfrft_denoise();
    d->cache = c;
    d->n = c->n;
    d->ch = channels;
    d->l = c->l;
    const int64_t cnt = d->n * channels;
    d->cpad = cnt + (cnt & 1);  // even: 16-byte aligned blocks
    d->cplx = !c->real;
    d->loss_on_real = loss_on_real != 0;
    const size_t blk = (size_t)d->cpad * 8, T = 2 * (size_t)d->l + 1, np = (size_t)d->n + 1;
    int rc = FGFRFT_OK;
    if (d->cplx) {  // complex blocks (the exact backend's buffers), [Q | dQ] complex, a ones diagonal
        const size_t cb = (size_t)cnt * 16;
        if (d->xytil.ensure(cb) || d->xu.ensure(cb) || d->xb.ensure(cb) || d->xw.ensure(cb) || d->xcot.ensure(cb) ||
            d->xvhr.ensure(cb) || d->xfar.ensure(cb) || d->xq.ensure(cb) || d->xt.ensure(cb) ||
            d->xph.ensure((size_t)d->n * 16))
            rc = fail(FGFRFT_CAPACITY, "denoise: device allocation failed");
    }
    if (rc != FGFRFT_OK || d->y.ensure(blk) || d->x.ensure(blk) ||
        d->qd.ensure(2 * (size_t)d->n * d->n * (d->cplx ? 16 : 8)) || d->uu.ensure(2 * blk) ||
        d->ww.ensure(2 * blk) || d->qr.ensure(blk) ||
        d->v.ensure(blk) || d->r.ensure(blk) || d->params.ensure(np * 8) || d->grad.ensure(np * 8) ||
        d->adam.ensure(2 * np * 8) || d->tab.ensure(4 * T * 8) || d->part.ensure(dn_part_elems() * 8) ||
        d->scal.ensure(8 * 8) || d->best.ensure((np + 1) * 8) || d->flag.ensure(4 * sizeof(int)))
        rc = fail(FGFRFT_CAPACITY, "denoise: device allocation failed");
    if (rc == FGFRFT_OK) {
        cudaMemsetAsync(d->y.p, 0, blk, c->stream);
        cudaMemsetAsync(d->x.p, 0, blk, c->stream);
        if (cudaMemcpyAsync(d->y.p, y, (size_t)cnt * 8, cudaMemcpyHostToDevice, c->stream) ||
            cudaMemcpyAsync(d->x.p, x_ref, (size_t)cnt * 8, cudaMemcpyHostToDevice, c->stream))
            rc = fail(FGFRFT_CUDA, "denoise: upload failed");
    }
    if (rc == FGFRFT_OK && d->cplx) {  // y as complex; the all-ones diagonal for dnx_grad
        std::vector<double2> ones((size_t)d->n, make_double2(1.0, 0.0));
        if (launch_real_to_cplx(d->y.as<double>(), cnt, d->xytil.p, c->stream) ||
            cudaMemcpyAsync(d->xph.p, ones.data(), ones.size() * 16, cudaMemcpyHostToDevice, c->stream) ||
            cudaStreamSynchronize(c->stream))
            rc = fail(FGFRFT_CUDA, "denoise: setup failed");
        g_launches += 1;
    }
    if (rc == FGFRFT_OK && cudaStreamSynchronize(c->stream) != cudaSuccess)
        rc = fail(FGFRFT_CUDA, "denoise: setup failed");
    if (rc != FGFRFT_OK) {
        fgfrft_denoise_destroy(d);
        return rc;
    }
    *out = d;
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_denoise_destroy(fgfrft_denoise* d) {
    if (!d) return FGFRFT_OK;
    if (d->cache || d->spec) {
        DeviceGuard dg(dn_device(d));
        cudaStreamSynchronize(dn_stream(d));
    }
    for (DevBuf* b : {&d->y, &d->x, &d->qd, &d->uu, &d->ww, &d->qr, &d->v, &d->r, &d->params,
                      &d->grad, &d->adam, &d->tab, &d->part, &d->scal, &d->best, &d->traj, &d->flag, &d->xytil,
                      &d->xu, &d->xb, &d->xw, &d->xcot, &d->xvhr, &d->xfar, &d->xq, &d->xt, &d->xph})
        b->release();
    delete d;
    return FGFRFT_OK;
}

int fgfrft_denoise_eval(fgfrft_denoise* d, double alpha, const double* h, double* loss, double* grad_alpha,
                        double* grad_h) {
    FGB_GUARD_BEGIN
    if (int st = check_denoise(d)) return st;
    if (!h) return fail(FGFRFT_PARAMETER, "null filter");
    std::lock_guard<std::mutex> lk(dn_mutex(d));
    DeviceGuard dg(dn_device(d));
    cudaStream_t st = dn_stream(d);
    double* params = d->params.as<double>();
    FGB_CUDA(cudaMemcpyAsync(params, &alpha, 8, cudaMemcpyHostToDevice, st));
    FGB_CUDA(cudaMemcpyAsync(params + 1, h, (size_t)d->n * 8, cudaMemcpyHostToDevice, st));
    FGB_CUDA(cudaMemsetAsync(d->flag.p, 0, sizeof(int), st));
    double* sl = d->scal.as<double>();
    if (int e = denoise_eval_device(d, params, sl, d->grad.as<double>())) return e;
    std::vector<double> g((size_t)d->n + 1);
    double lv = 0.0;
    FGB_CUDA(cudaMemcpyAsync(&lv, sl, 8, cudaMemcpyDeviceToHost, st));
    FGB_CUDA(cudaMemcpyAsync(g.data(), d->grad.p, g.size() * 8, cudaMemcpyDeviceToHost, st));
    FGB_CUDA(cudaStreamSynchronize(st));
    if (loss) *loss = lv;
    if (grad_alpha) *grad_alpha = g[0];
    if (grad_h) std::memcpy(grad_h, g.data() + 1, (size_t)d->n * 8);
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_denoise_fit(fgfrft_denoise* d, int epochs, double lr, double init_alpha, double* traj_loss,
                       double* traj_alpha, double* alpha_best, double* h_best, double* loss_best, int* best_epoch,
                       double* reconstruction) {
    FGB_GUARD_BEGIN
    if (int st = check_denoise(d)) return st;
    if (epochs < 1) return fail(FGFRFT_PARAMETER, "DenoiseConfig: epochs must be >= 1");
    if (!(lr > 0.0)) return fail(FGFRFT_PARAMETER, "DenoiseConfig: lr must be positive");
    std::lock_guard<std::mutex> lk(dn_mutex(d));
    DeviceGuard dg(dn_device(d));
    cudaStream_t cst = dn_stream(d);
    const int np = (int)d->n + 1;
    FGB_CUDA(d->traj.ensure((size_t)2 * (epochs + 1) * 8));
    double* params = d->params.as<double>();
    double* m = d->adam.as<double>();
    double* best = d->best.as<double>();
    double* sl = d->scal.as<double>();
    int* bep = d->flag.as<int>() + 1;
    {  // params = [init_alpha, 1 .. 1] (learn.hpp:475-478); Adam moments zero; best loss = +inf
        std::vector<double> p0((size_t)np, 1.0);
        p0[0] = init_alpha;
        const double inf = std::numeric_limits<double>::infinity();
        FGB_CUDA(cudaMemcpyAsync(params, p0.data(), (size_t)np * 8, cudaMemcpyHostToDevice, cst));
        FGB_CUDA(cudaMemsetAsync(m, 0, (size_t)2 * np * 8, cst));
        FGB_CUDA(cudaMemcpyAsync(best, &inf, 8, cudaMemcpyHostToDevice, cst));
        const int fl0[4] = {0, 0, std::numeric_limits<int>::max(), std::numeric_limits<int>::max()};
        FGB_CUDA(cudaMemcpyAsync(d->flag.p, fl0, sizeof fl0, cudaMemcpyHostToDevice, cst));
        FGB_CUDA(cudaStreamSynchronize(cst));  // p0 / inf / fl0 are host stack buffers
    }
    for (int e = 0; e <= epochs; ++e) {  // the final evaluation (e == epochs) is not checked
        if (int st = denoise_eval_device(d, params, sl, d->grad.as<double>(), e < epochs ? e : -1)) return st;
        FGB_LAUNCH(launch_dn_track(sl, params, np, e, d->traj.as<double>(), best, bep, cst), 1);
        if (e < epochs) FGB_LAUNCH(launch_dn_adam(params, m, m + np, d->grad.as<double>(), np, e + 1, lr, cst), 1);
    }
    int flags[4] = {0, 0, 0, 0};
    FGB_CUDA(cudaMemcpyAsync(flags, d->flag.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, cst));
    std::vector<double> tr((size_t)2 * (epochs + 1)), bb((size_t)np + 1);
    FGB_CUDA(cudaMemcpyAsync(tr.data(), d->traj.p, tr.size() * 8, cudaMemcpyDeviceToHost, cst));
    FGB_CUDA(cudaMemcpyAsync(bb.data(), best, bb.size() * 8, cudaMemcpyDeviceToHost, cst));
    FGB_CUDA(cudaStreamSynchronize(cst));
    // the reference loop stops at the first failing check: loss of epoch e, then the Adam step's
    // gradient check (step e + 1)
    if ((flags[0] & 1) && (!(flags[0] & 2) || flags[2] <= flags[3])) {
        std::ostringstream msg;
        msg << "denoise: non-finite loss at epoch " << flags[2];
        return fail(FGFRFT_OPTIMIZER, msg.str());
    }
    if (flags[0] & 2) {
        std::ostringstream msg;
        msg << "adam_step: non-finite gradient at step " << flags[3] + 1;
        return fail(FGFRFT_OPTIMIZER, msg.str());
    }
    for (int e = 0; e <= epochs; ++e) {
        if (traj_loss) traj_loss[e] = tr[2 * e];
        if (traj_alpha) traj_alpha[e] = tr[2 * e + 1];
    }
    if (loss_best) *loss_best = bb[0];
    if (alpha_best) *alpha_best = bb[1];
    if (h_best) std::memcpy(h_best, bb.data() + 2, (size_t)d->n * 8);
    if (best_epoch) *best_epoch = flags[1];
    if (reconstruction) {  // real part of w at the best parameters (learn.hpp:514)
        FGB_CUDA(cudaMemcpyAsync(params, best + 1, (size_t)np * 8, cudaMemcpyDeviceToDevice, cst));
        if (int st = denoise_eval_device(d, params, sl, d->grad.as<double>())) return st;
        const void* src = d->ww.p;
        if (d->exact || d->cplx) {  // Re w
            FGB_LAUNCH(launch_real_part(d->xw.p, d->xt.p, d->n * d->ch, cst), 1);
            src = d->xt.p;
        }
        FGB_CUDA(cudaMemcpyAsync(reconstruction, src, (size_t)d->n * d->ch * 8, cudaMemcpyDeviceToHost, cst));
        FGB_CUDA(cudaStreamSynchronize(cst));
    }
    return FGFRFT_OK;
    FGB_GUARD_END
}

}  // extern "C"

// ------------------------------------------------------------------ exact denoise backend
//
// learn.hpp:205-289 (ExactDenoiseEngine) on the device spectrum: per evaluation six DMMA ZGEMMs
// with V / V^H (u, b, w, V^H r, F^a r, q) around diagonal scalings (denoise.cu dnx_*), the loss
// and both gradients reduced in a fixed order; the Adam loop / tracking is the fast backend's.

namespace fgbi {

cudaStream_t dn_stream(const fgfrft_denoise* d) { return d->exact ? d->spec->stream : d->cache->stream; }
std::mutex& dn_mutex(fgfrft_denoise* d) { return d->exact ? d->spec->mu : d->cache->mu; }
int dn_device(const fgfrft_denoise* d) { return d->exact ? d->spec->device : d->cache->device; }

int denoise_exact_eval(fgfrft_denoise* d, const double* params, double* loss, double* grad, int epoch) {
    fgfrft_spectrum* s = d->spec;
    cudaStream_t st = s->stream;
    const int n = (int)d->n, ch = (int)d->ch;
    const int64_t cnt = (int64_t)n * ch;
    const double* h = params + 1;
    double2* ph = d->xph.as<double2>();
    double2* jtp = ph + n;
    double2* jtc = ph + 2 * n;
    auto zg = [&](bool adj, const void* b, void* c) -> int {  // c = V b or V^H b
        return zgemm_auto(adj ? 2 : 0, 0, n, ch, n, s->v.p, n, 0, b, n, 0, c, n, 0, 1, st);
    };
    FGB_LAUNCH(launch_dnx_phase(params, s->theta.as<double>(), n, ph, jtp, jtc, st), 1);
    FGB_LAUNCH(launch_dnx_rowscale(d->xytil.p, ph, nullptr, false, n, cnt, d->xt.p, st), 1);
    if (int e = zg(false, d->xt.p, d->xu.p)) return e;                          // u = V (phase o ytil)
    FGB_LAUNCH(launch_dnx_rowscale(d->xu.p, nullptr, h, false, n, cnt, d->xt.p, st), 1);
    if (int e = zg(true, d->xt.p, d->xb.p)) return e;                           // b = V^H (h o u)
    FGB_LAUNCH(launch_dnx_rowscale(d->xb.p, ph, nullptr, true, n, cnt, d->xt.p, st), 1);
    if (int e = zg(false, d->xt.p, d->xw.p)) return e;                          // w = V (conj(phase) o b)
    double* part = d->part.as<double>();
    FGB_LAUNCH(launch_dnx_cot(d->xw.p, d->x.as<double>(), cnt, d->loss_on_real, d->xcot.p, part, st), 1);
    if (int e = zg(true, d->xcot.p, d->xvhr.p)) return e;                       // V^H r
    FGB_LAUNCH(launch_dnx_rowscale(d->xvhr.p, ph, nullptr, false, n, cnt, d->xt.p, st), 1);
    if (int e = zg(false, d->xt.p, d->xfar.p)) return e;                        // F^a r
    FGB_LAUNCH(launch_dnx_rowscale(d->xytil.p, jtp, nullptr, false, n, cnt, d->xt.p, st), 1);
    if (int e = zg(false, d->xt.p, d->xq.p)) return e;                          // q = V (j theta phase o ytil)
    FGB_LAUNCH(launch_dnx_grad(d->xfar.p, d->xu.p, d->xvhr.p, d->xb.p, jtc, d->xq.p, h, n, ch, grad + 1, part, st),
               1);
    FGB_LAUNCH(launch_dn_finish(part, loss, grad, n, d->flag.as<int>(), epoch, st), 1);
    return FGFRFT_OK;
}

}  // namespace fgbi

extern "C" {

int fgfrft_denoise_create_exact(fgfrft_spectrum* spec, const double* y, const double* x_ref, int64_t channels,
                                int loss_on_real, fgfrft_denoise** out) {
    FGB_GUARD_BEGIN
    if (!out) return fail(FGFRFT_PARAMETER, "null output handle pointer");
    *out = nullptr;
    if (int st = check_spectrum(spec)) return st;
    if (channels < 1) return fail(FGFRFT_SHAPE, "denoise: need at least one channel");
    if (!y || !x_ref) return fail(FGFRFT_PARAMETER, "null signal buffer");
    std::lock_guard<std::mutex> lk(spec->mu);
    DeviceGuard dg(spec->device);
    auto* d = new fgfrft_denoise();
    d->spec = spec;
    d->exact = true;
    d->loss_on_real = loss_on_real != 0;
    d->n = spec->n;
    d->ch = channels;
    const int64_t cnt = d->n * channels;
    d->cpad = cnt;
    const size_t cb = (size_t)cnt * 16, np = (size_t)d->n + 1;
    cudaStream_t st = spec->stream;
    int rc = FGFRFT_OK;
    if (d->y.ensure(cnt * 8) || d->x.ensure(cnt * 8) || d->xytil.ensure(cb) || d->xu.ensure(cb) || d->xb.ensure(cb) ||
        d->xw.ensure(cb) || d->xcot.ensure(cb) || d->xvhr.ensure(cb) || d->xfar.ensure(cb) || d->xq.ensure(cb) ||
        d->xt.ensure(cb) || d->xph.ensure((size_t)3 * d->n * 16) || d->params.ensure(np * 8) ||
        d->grad.ensure(np * 8) || d->adam.ensure(2 * np * 8) || d->part.ensure(dn_part_elems() * 8) ||
        d->scal.ensure(8 * 8) || d->best.ensure((np + 1) * 8) || d->flag.ensure(4 * sizeof(int)))
        rc = fail(FGFRFT_CAPACITY, "denoise: device allocation failed");
    if (rc == FGFRFT_OK && (cudaMemcpyAsync(d->y.p, y, (size_t)cnt * 8, cudaMemcpyHostToDevice, st) ||
                            cudaMemcpyAsync(d->x.p, x_ref, (size_t)cnt * 8, cudaMemcpyHostToDevice, st)))
        rc = fail(FGFRFT_CUDA, "denoise: upload failed");
    if (rc == FGFRFT_OK) {  // ytil = V^H y (learn.hpp:210), y promoted to complex
        if (launch_real_to_cplx(d->y.as<double>(), cnt, d->xt.p, st) ||
            launch_zgemm((int)d->n, (int)channels, (int)d->n, spec->v.p, d->n, 0, true, d->xt.p, d->n, 0, false,
                         d->xytil.p, d->n, 0, 1, false, st) ||
            cudaStreamSynchronize(st))
            rc = fail(FGFRFT_CUDA, "denoise: setup failed");
        g_launches += 2;
    }
    if (rc != FGFRFT_OK) {
        fgfrft_denoise_destroy(d);
        return rc;
    }
    *out = d;
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_denoise_reconstruct(fgfrft_denoise* d, double alpha, const double* h, double* out) {
    FGB_GUARD_BEGIN
    if (int st = check_denoise(d)) return st;
    if (!h || !out) return fail(FGFRFT_PARAMETER, "null buffer");
    std::lock_guard<std::mutex> lk(dn_mutex(d));
    DeviceGuard dg(dn_device(d));
    cudaStream_t st = dn_stream(d);
    double* params = d->params.as<double>();
    FGB_CUDA(cudaMemcpyAsync(params, &alpha, 8, cudaMemcpyHostToDevice, st));
    FGB_CUDA(cudaMemcpyAsync(params + 1, h, (size_t)d->n * 8, cudaMemcpyHostToDevice, st));
    if (int e = denoise_eval_device(d, params, d->scal.as<double>(), d->grad.as<double>())) return e;
    const void* src = d->ww.p;
    if (d->exact || d->cplx) {  // Re w (learn.hpp:232-234, 405-408)
        FGB_LAUNCH(launch_real_part(d->xw.p, d->xt.p, d->n * d->ch, st), 1);
        src = d->xt.p;
    }
    FGB_CUDA(cudaMemcpyAsync(out, src, (size_t)d->n * d->ch * 8, cudaMemcpyDeviceToHost, st));
    FGB_CUDA(cudaStreamSynchronize(st));
    return FGFRFT_OK;
    FGB_GUARD_END
}

}  // extern "C"
