// denoise.cu -- device kernels of the GPU-resident denoising learner.
//
// Restates the reference's fast matrix-free denoise engine (learn.hpp:291-413, real F) and its
// training loop (learn.hpp:471-516, Adam of adam.hpp:34-53) on the device. One evaluation at
// (alpha, h), with spow_m = F^m y precomputed once and every "F^m applied to a block" done as
// ONE INT8 power-product GEMM over the stacked cache (ozgemm.cu):
//   u = sum c_m spow_m,  du = sum c'_m spow_m               (combine pass over spow, 2 rows)
//   v = h o u,  tpow_m = F^m v                               (power products)
//   w = Q^H v = sum c_-m tpow_m,  dqh_v = sum c'_-m tpow_m   (combine pass over tpow, 2 rows)
//   r = w - x,  loss = |r|^2                                 (learn.hpp:392-404)
//   gpow_m = F^m r,  qr = sum c_m gpow_m                     (power products + combine)
//   grad_h = 2 rowsum(qr o u),  grad_alpha = 2 <r, dqh_v> + 2 <qr, h o du>   (learn.hpp:310-337)
// These kernels are the small pieces around the power products and the combinations.
#include "common.cuh"

namespace fgb {

// Coefficient tables from the device-resident alpha = params[0]:
//   tab[0][q] = c(alpha)[q],  tab[1][q] = c'(alpha)[q]                (spow / gpow passes)
//   tab[2][q] = c(alpha)[2L - q],  tab[3][q] = c'(alpha)[2L - q]      (tpow pass: c_-m, c'_-m)
__global__ void dn_coef_kernel(const double* __restrict__ params, int l, double* __restrict__ tab) {
    const int T = 2 * l + 1;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= T) return;
    const double a = params[0];
    const double x = a - (double)(q - l);
    const double xr = a - (double)(l - q);  // term 2L - q
    tab[q] = dsinc(x);
    tab[T + q] = dsinc_deriv(x);
    tab[2 * T + q] = dsinc(xr);
    tab[3 * T + q] = dsinc_deriv(xr);
}

// v[i + c n] = h[i] u[i + c n]
__global__ void dn_scale_kernel(const double* __restrict__ u, const double* __restrict__ h, double* __restrict__ v,
                                int n, int64_t count) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x)
        v[p] = h[p % n] * u[p];
}

__device__ __forceinline__ double block_sum256(double v, double* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];  // fixed order
    __syncthreads();
    return s;
}

constexpr int kDnBlocks = 2 * FGFRFT_SMS;

// r = w - x and per-block partial sums of r^2 (part[0][block])
__global__ void __launch_bounds__(256) dn_residual_kernel(const double* __restrict__ w, const double* __restrict__ x,
                                                          double* __restrict__ r, int64_t count,
                                                          double* __restrict__ part) {
    __shared__ double red[8];
    double acc = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x) {
        const double d = w[p] - x[p];
        r[p] = d;
        acc = fma(d, d, acc);
    }
    acc = block_sum256(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// grad_h[i] = 2 sum_c qr[i, c] u[i, c]; per-block partials of <r, dqh_v> + <qr, h o du>
__global__ void __launch_bounds__(256) dn_grad_kernel(const double* __restrict__ u, const double* __restrict__ du,
                                                      const double* __restrict__ h, const double* __restrict__ r,
                                                      const double* __restrict__ dqhv, const double* __restrict__ qr,
                                                      int n, int ch, double* __restrict__ grad_h,
                                                      double* __restrict__ part) {
    __shared__ double red[8];
    const int64_t count = (int64_t)n * ch;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int c = 0; c < ch; ++c) acc = fma(qr[i + (int64_t)c * n], u[i + (int64_t)c * n], acc);
        grad_h[i] = 2.0 * acc;
    }
    double acc = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x)
        acc = fma(r[p], dqhv[p], fma(qr[p], h[p % n] * du[p], acc));
    acc = block_sum256(acc, red);
    if (threadIdx.x == 0) part[kDnBlocks + blockIdx.x] = acc;
}

// loss = sum part[0][:], grad_alpha = 2 sum part[1][:] (fixed order). For a training epoch
// (epoch >= 0) a non-finite loss / gradient sets flag[0] bit 1 / 2 and the first such epoch in
// flag[2] / flag[3] (learn.hpp:499-505 and adam.hpp:36-42 checks, evaluated after the loop).
__global__ void dn_finish_kernel(const double* __restrict__ part, double* __restrict__ loss,
                                 double* __restrict__ grad, int n, int* __restrict__ flag, int epoch) {
    __shared__ double red[8];
    double a = 0.0, g = 0.0;
    for (int b = threadIdx.x; b < kDnBlocks; b += 256) {
        a += part[b];
        g += part[kDnBlocks + b];
    }
    a = block_sum256(a, red);
    g = block_sum256(g, red);
    if (threadIdx.x == 0) {
        *loss = a;
        grad[0] = 2.0 * g;
        if (epoch >= 0 && !isfinite(a)) {
            atomicOr(flag, 1);
            atomicMin(flag + 2, epoch);
        }
    }
    if (epoch < 0) return;
    for (int i = threadIdx.x; i < n + 1; i += 256)
        if (!isfinite(grad[i])) {
            atomicOr(flag, 2);
            atomicMin(flag + 3, epoch);
        }
}

// trajectory[epoch] = (loss, alpha); best <- params when loss improves (learn.hpp:483-491)
__global__ void dn_track_kernel(const double* __restrict__ loss, const double* __restrict__ params, int np, int epoch,
                                double* __restrict__ traj, double* __restrict__ best, int* __restrict__ best_epoch) {
    __shared__ bool better;
    if (threadIdx.x == 0) {
        traj[2 * epoch] = *loss;
        traj[2 * epoch + 1] = params[0];
        better = *loss < best[0];  // best[0] = best loss, best[1..np] = params
        if (better) {
            best[0] = *loss;
            *best_epoch = epoch;
        }
    }
    __syncthreads();
    if (better)
        for (int i = threadIdx.x; i < np; i += blockDim.x) best[1 + i] = params[i];
}

// Bias-corrected Adam (adam.hpp:34-53); state = [m | v], step = the new step count.
__global__ void dn_adam_kernel(double* __restrict__ params, double* __restrict__ m, double* __restrict__ v,
                               const double* __restrict__ grad, int np, int64_t step, double lr, double beta1,
                               double beta2, double eps) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    const double g = grad[i];
    const double mi = beta1 * m[i] + (1.0 - beta1) * g;
    const double vi = beta2 * v[i] + (1.0 - beta2) * (g * g);
    m[i] = mi;
    v[i] = vi;
    const double c1 = 1.0 - pow(beta1, (double)step);
    const double c2 = 1.0 - pow(beta2, (double)step);
    params[i] = params[i] - lr * (mi / c1) / (sqrt(vi / c2) + eps);
}

cudaError_t launch_dn_coef(const double* params, int l, double* tab, cudaStream_t st) {
    dn_coef_kernel<<<(2 * l + 1 + 127) / 128, 128, 0, st>>>(params, l, tab);
    return cudaGetLastError();
}
cudaError_t launch_dn_scale(const double* u, const double* h, double* v, int n, int64_t count, cudaStream_t st) {
    dn_scale_kernel<<<kDnBlocks, 256, 0, st>>>(u, h, v, n, count);
    return cudaGetLastError();
}
cudaError_t launch_dn_residual(const double* w, const double* x, double* r, int64_t count, double* part,
                               cudaStream_t st) {
    dn_residual_kernel<<<kDnBlocks, 256, 0, st>>>(w, x, r, count, part);
    return cudaGetLastError();
}
cudaError_t launch_dn_grad(const double* u, const double* du, const double* h, const double* r, const double* dqhv,
                           const double* qr, int n, int ch, double* grad, double* part, double* loss, int* flag,
                           int epoch, cudaStream_t st) {
    dn_grad_kernel<<<kDnBlocks, 256, 0, st>>>(u, du, h, r, dqhv, qr, n, ch, grad + 1, part);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    dn_finish_kernel<<<1, 256, 0, st>>>(part, loss, grad, n, flag, epoch);
    return cudaGetLastError();
}
cudaError_t launch_dn_track(const double* loss, const double* params, int np, int epoch, double* traj, double* best,
                            int* best_epoch, cudaStream_t st) {
    dn_track_kernel<<<1, 256, 0, st>>>(loss, params, np, epoch, traj, best, best_epoch);
    return cudaGetLastError();
}
cudaError_t launch_dn_adam(double* params, double* m, double* v, const double* grad, int np, int64_t step, double lr,
                           cudaStream_t st) {
    dn_adam_kernel<<<(np + 255) / 256, 256, 0, st>>>(params, m, v, grad, np, step, lr, 0.9, 0.999, 1e-8);
    return cudaGetLastError();
}
size_t dn_part_elems() { return 2 * (size_t)kDnBlocks; }

// ---------------------------------------------------------------- exact backend (learn.hpp:205-289)
//
// F^a = V diag(e^{j a theta}) V^H on the device spectrum; every product with V / V^H is a DMMA
// ZGEMM (capi.cu), these kernels are the diagonal scalings and the reductions around them. All
// blocks are n x ch complex128, column-major; row i of a spectral-domain block is eigen index i.

// phase = e^{j a theta}, jtp = j theta e^{j a theta}, jtc = -j theta e^{-j a theta}; a = params[0]
__global__ void dnx_phase_kernel(const double* __restrict__ params, const double* __restrict__ theta, int n,
                                 double2* __restrict__ phase, double2* __restrict__ jtp, double2* __restrict__ jtc) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double th = theta[k];
    double s, c;
    sincos(params[0] * th, &s, &c);
    phase[k] = make_double2(c, s);
    jtp[k] = make_double2(-th * s, th * c);  // (j th)(c + j s)
    jtc[k] = make_double2(-th * s, -th * c); // (-j th)(c - j s)
}

// dst[i, c] = d[i] src[i, c] (conj_d: conj(d[i])); real_h: d is the real filter h = params + 1
__global__ void dnx_rowscale_kernel(const double2* __restrict__ src, const double2* __restrict__ d,
                                    const double* __restrict__ h, bool conj_d, int n, int64_t count,
                                    double2* __restrict__ dst) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(p % n);
        const double2 v = src[p];
        if (h) {
            dst[p] = make_double2(h[i] * v.x, h[i] * v.y);
        } else {
            const double dx = d[i].x, dy = conj_d ? -d[i].y : d[i].y;
            dst[p] = make_double2(fma(dx, v.x, -dy * v.y), fma(dx, v.y, dy * v.x));
        }
    }
}

// cot = w - x (or Re w - x with loss_on_real), part[blk] = sum |cot|^2
__global__ void __launch_bounds__(256) dnx_cot_kernel(const double2* __restrict__ w, const double* __restrict__ x,
                                                      int64_t count, bool real_loss, double2* __restrict__ cot,
                                                      double* __restrict__ part) {
    __shared__ double red[8];
    double acc = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x) {
        const double2 r = make_double2(w[p].x - x[p], real_loss ? 0.0 : w[p].y);
        cot[p] = r;
        acc = fma(r.x, r.x, fma(r.y, r.y, acc));
    }
    acc = block_sum256(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// grad_h[i] = 2 sum_c Re(conj(far[i, c]) u[i, c]);
// part[kDnBlocks + blk] = sum Re(conj(vhr) jtc o b) + Re(conj(far) h o q)  (grad_alpha / 2)
__global__ void __launch_bounds__(256) dnx_grad_kernel(const double2* __restrict__ far, const double2* __restrict__ u,
                                                       const double2* __restrict__ vhr, const double2* __restrict__ b,
                                                       const double2* __restrict__ jtc, const double2* __restrict__ q,
                                                       const double* __restrict__ h, int n, int ch,
                                                       double* __restrict__ grad_h, double* __restrict__ part) {
    __shared__ double red[8];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int c = 0; c < ch; ++c) {
            const double2 f = far[i + (int64_t)c * n], uu = u[i + (int64_t)c * n];
            acc = fma(f.x, uu.x, fma(f.y, uu.y, acc));
        }
        grad_h[i] = 2.0 * acc;
    }
    const int64_t count = (int64_t)n * ch;
    double acc = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(p % n);
        const double2 t = make_double2(fma(jtc[i].x, b[p].x, -jtc[i].y * b[p].y), fma(jtc[i].x, b[p].y, jtc[i].y * b[p].x));
        acc = fma(vhr[p].x, t.x, fma(vhr[p].y, t.y, acc));
        const double2 hq = make_double2(h[i] * q[p].x, h[i] * q[p].y);
        acc = fma(far[p].x, hq.x, fma(far[p].y, hq.y, acc));
    }
    acc = block_sum256(acc, red);
    if (threadIdx.x == 0) part[kDnBlocks + blockIdx.x] = acc;
}

cudaError_t launch_dnx_phase(const double* params, const double* theta, int n, void* phase, void* jtp, void* jtc,
                             cudaStream_t st) {
    dnx_phase_kernel<<<(n + 127) / 128, 128, 0, st>>>(params, theta, n, (double2*)phase, (double2*)jtp,
                                                      (double2*)jtc);
    return cudaGetLastError();
}
cudaError_t launch_dnx_rowscale(const void* src, const void* d, const double* h, bool conj_d, int n, int64_t count,
                                void* dst, cudaStream_t st) {
    dnx_rowscale_kernel<<<kDnBlocks, 256, 0, st>>>((const double2*)src, (const double2*)d, h, conj_d, n, count,
                                                   (double2*)dst);
    return cudaGetLastError();
}
cudaError_t launch_dnx_cot(const void* w, const double* x, int64_t count, bool real_loss, void* cot, double* part,
                           cudaStream_t st) {
    dnx_cot_kernel<<<kDnBlocks, 256, 0, st>>>((const double2*)w, x, count, real_loss, (double2*)cot, part);
    return cudaGetLastError();
}
cudaError_t launch_dnx_grad(const void* far, const void* u, const void* vhr, const void* b, const void* jtc,
                            const void* q, const double* h, int n, int ch, double* grad_h, double* part,
                            cudaStream_t st) {
    dnx_grad_kernel<<<kDnBlocks, 256, 0, st>>>((const double2*)far, (const double2*)u, (const double2*)vhr,
                                               (const double2*)b, (const double2*)jtc, (const double2*)q, h, n, ch,
                                               grad_h, part);
    return cudaGetLastError();
}
cudaError_t launch_dn_finish(const double* part, double* loss, double* grad, int n, int* flag, int epoch,
                             cudaStream_t st) {
    dn_finish_kernel<<<1, 256, 0, st>>>(part, loss, grad, n, flag, epoch);
    return cudaGetLastError();
}

}  // namespace fgb
