// spectral.cu -- device kernels of the exact-GFRFT path and of the cascaded
// order learner (rank 2).
//
// Exact operator (spectral.hpp:158-174): F^a = V diag(e^{j a theta}) V^H and
// dF^a/da = V diag(j theta e^{j a theta}) V^H, done as one column scaling (spec_scale_kernel) and
// one DMMA complex GEMM W V^H (zgemm.cu). Eigendecomposition of a unitary F (spectral.hpp:55-155):
// the Hermitian part goes to cuSOLVER (capi.cu), the pieces around it are here -- Hermitian parts,
// cluster Gram blocks W_c^H B W_c, block-diagonal column mixing, Rayleigh quotients.
// Cascade (learn.hpp:72-97): residual / squared norm and Re<M, dQ> reductions in a fixed order.
#include <algorithm>

#include "common.cuh"

namespace fgb {

constexpr int kSpRedBlocks = 2 * FGFRFT_SMS;
constexpr int kSpRedThreads = 256;

// A = (F + F^H)/2 (real F: the real symmetric part, stored as doubles for Dsyevd),
// Bh = -i/2 (F - F^H)   (spectral.hpp:84-89, 101-104; for real F Bh = -i (F - F^T)/2)
__global__ void herm_parts_kernel(const double2* __restrict__ f, int n, bool real, void* __restrict__ a,
                                  double2* __restrict__ bh) {
    const int64_t count = (int64_t)n * n;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(p % n), j = (int)(p / n);
        const double2 fij = f[p], fji = f[j + (int64_t)i * n];
        if (real) {
            static_cast<double*>(a)[p] = 0.5 * (fij.x + fji.x);
            bh[p] = make_double2(0.0, -(0.5 * (fij.x - fji.x)));
        } else {
            static_cast<double2*>(a)[p] = make_double2(0.5 * (fij.x + fji.x), 0.5 * (fij.y - fji.y));
            const double dx = fij.x - fji.x, dy = fij.y + fji.y;  // F - F^H
            bh[p] = make_double2(0.5 * dy, -0.5 * dx);
        }
    }
}

__global__ void real_to_cplx_kernel(const double* __restrict__ src, int64_t count, double2* __restrict__ dst) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x)
        dst[p] = make_double2(src[p], 0.0);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // conj(a) b
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
}

// out[:, c] = sum_i in[:, lo_c + i] U_c[i, c - lo_c]: the cluster rotations of spectral.hpp:62-64.
// colinfo[3c..3c+2] = (lo, k, offset of the column-major k x k block in u).
__global__ void blockdiag_kernel(const double2* __restrict__ in, int n, const int* __restrict__ colinfo,
                                 const double2* __restrict__ u, double2* __restrict__ out) {
    const int c = blockIdx.y;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int lo = colinfo[3 * c], k = colinfo[3 * c + 1], off = colinfo[3 * c + 2];
    const int j = c - lo;
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < k; ++i) {
        const double2 w = in[r + (int64_t)(lo + i) * n], s = u[off + i + j * k];
        acc.x += w.x * s.x - w.y * s.y;
        acc.y += w.x * s.y + w.y * s.x;
    }
    out[r + (int64_t)c * n] = acc;
}

// out[e] = sum_r conj(W[r, pa_e]) T[r, pb_e] (one warp per entry, fixed-order reduction):
// the cluster restrictions W_c^H Bh W_c (spectral.hpp:61) and the Rayleigh quotients v^H F v (:67).
__global__ void col_pair_dot_kernel(const double2* __restrict__ w, const double2* __restrict__ t, int n,
                                    const int* __restrict__ pairs, int count, double2* __restrict__ out) {
    const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (e >= count) return;
    const double2* a = w + (int64_t)pairs[2 * e] * n;
    const double2* b = t + (int64_t)pairs[2 * e + 1] * n;
    double2 acc = make_double2(0.0, 0.0);
    for (int r = lane; r < n; r += 32) {
        const double2 p = cmulc(a[r], b[r]);
        acc.x += p.x;
        acc.y += p.y;
    }
    for (int o = 16; o; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) out[e] = acc;
}

// dst[:, k] = src[:, perm[k]]
__global__ void gather_cols_kernel(const double2* __restrict__ src, int n, const int* __restrict__ perm,
                                   double2* __restrict__ dst) {
    const int c = blockIdx.y;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) dst[r + (int64_t)c * n] = src[r + (int64_t)perm[c] * n];
}

__device__ __forceinline__ double block_sum(double v, double* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < kSpRedThreads / 32; ++w) s += red[w];
    __syncthreads();
    return s;
}

// part[blk] = sum |FW[:, c] - e^{j theta_c} W[:, c]|^2, part[G + blk] = sum |F|^2 (spectral.hpp:141-146)
__global__ void __launch_bounds__(kSpRedThreads) eig_residual_kernel(const double2* __restrict__ fw,
                                                                     const double2* __restrict__ w,
                                                                     const double* __restrict__ theta,
                                                                     const double2* __restrict__ f, int n,
                                                                     double* __restrict__ part) {
    __shared__ double red[kSpRedThreads / 32];
    const int64_t count = (int64_t)n * n;
    double acc = 0.0, fn = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(p / n);
        double s, co;
        sincos(theta[c], &s, &co);
        const double2 v = cmul(make_double2(co, s), w[p]);
        const double dx = fw[p].x - v.x, dy = fw[p].y - v.y;
        acc = fma(dx, dx, fma(dy, dy, acc));
        fn = fma(f[p].x, f[p].x, fma(f[p].y, f[p].y, fn));
    }
    acc = block_sum(acc, red);
    fn = block_sum(fn, red);
    if (threadIdx.x == 0) {
        part[blockIdx.x] = acc;
        part[gridDim.x + blockIdx.x] = fn;
    }
}

// W_a[:, k] = V[:, k] d_a(k): d = e^{j a theta_k} (which 0) or j theta_k e^{j a theta_k} (which 1)
// (spectral.hpp:160-161, 171-172; std::polar(1, x) = (cos x, sin x))
__global__ void spec_scale_kernel(const double2* __restrict__ v, const double* __restrict__ theta,
                                  const double* __restrict__ alphas, int na, int which, int n,
                                  double2* __restrict__ w) {
    const int64_t count = (int64_t)n * n;
    const int a = blockIdx.y;
    const double al = alphas[a];
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(p / n);
        const double th = theta[k];
        double s, c;
        sincos(al * th, &s, &c);
        const double2 d = which == 0 ? make_double2(c, s) : make_double2(-th * s, th * c);
        w[(int64_t)a * count + p] = cmul(v[p], d);
    }
}

// ---- cascade reductions (learn.hpp:85-92)

// b = y - t, part[blk] = sum |b|^2 (REAL_Y: y is a real n x n matrix, the real-F fast backend)
template <bool REAL_Y>
__global__ void __launch_bounds__(kSpRedThreads) cdiff_sq_kernel(const void* __restrict__ yv,
                                                                 const double2* __restrict__ t, int64_t count,
                                                                 double2* __restrict__ b, double* __restrict__ part) {
    __shared__ double red[kSpRedThreads / 32];
    double acc = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x) {
        const double2 y = REAL_Y ? make_double2(static_cast<const double*>(yv)[p], 0.0)
                                 : static_cast<const double2*>(yv)[p];
        const double2 d = make_double2(y.x - t[p].x, y.y - t[p].y);
        b[p] = d;
        acc = fma(d.x, d.x, fma(d.y, d.y, acc));
    }
    acc = block_sum(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// part[blk] = Re sum conj(m) o d (REAL_D: d is real)
template <bool REAL_D>
__global__ void __launch_bounds__(kSpRedThreads) cre_dot_kernel(const double2* __restrict__ m,
                                                                const void* __restrict__ dv, int64_t count,
                                                                double* __restrict__ part) {
    __shared__ double red[kSpRedThreads / 32];
    double acc = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x) {
        if (REAL_D) {
            acc = fma(m[p].x, static_cast<const double*>(dv)[p], acc);
        } else {
            const double2 d = static_cast<const double2*>(dv)[p];
            acc = fma(m[p].x, d.x, fma(m[p].y, d.y, acc));
        }
    }
    acc = block_sum(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// part[blk] = sum a o b (real)
__global__ void __launch_bounds__(kSpRedThreads) rdot_kernel(const double* __restrict__ a,
                                                             const double* __restrict__ b, int64_t count,
                                                             double* __restrict__ part) {
    __shared__ double red[kSpRedThreads / 32];
    double acc = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x)
        acc = fma(a[p], b[p], acc);
    acc = block_sum(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// out[g] = scale_g * sum_b part[g * G + b] (fixed order), scale_0 = s0, scale_{g>0} = s1
__global__ void sum_parts_kernel(const double* __restrict__ part, int groups, double s0, double s1,
                                 double* __restrict__ out) {
    __shared__ double red[kSpRedThreads / 32];
    for (int g = 0; g < groups; ++g) {
        double acc = 0.0;
        for (int b = threadIdx.x; b < kSpRedBlocks; b += blockDim.x) acc += part[(size_t)g * kSpRedBlocks + b];
        acc = block_sum(acc, red);
        if (threadIdx.x == 0) out[g] = (g == 0 ? s0 : s1) * acc;
    }
}

// ---- launchers

size_t sp_part_elems() { return kSpRedBlocks; }

cudaError_t launch_herm_parts(const void* f, int n, bool real, void* a, void* bh, cudaStream_t st) {
    herm_parts_kernel<<<2 * FGFRFT_SMS * 4, 256, 0, st>>>((const double2*)f, n, real, a, (double2*)bh);
    return cudaGetLastError();
}
cudaError_t launch_real_to_cplx(const double* src, int64_t count, void* dst, cudaStream_t st) {
    real_to_cplx_kernel<<<2 * FGFRFT_SMS * 4, 256, 0, st>>>(src, count, (double2*)dst);
    return cudaGetLastError();
}
cudaError_t launch_blockdiag(const void* in, int n, const int* colinfo, const void* u, void* out, cudaStream_t st) {
    blockdiag_kernel<<<dim3((unsigned)((n + 127) / 128), (unsigned)n), 128, 0, st>>>(
        (const double2*)in, n, colinfo, (const double2*)u, (double2*)out);
    return cudaGetLastError();
}
cudaError_t launch_col_pair_dot(const void* w, const void* t, int n, const int* pairs, int count, void* out,
                                cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    col_pair_dot_kernel<<<(unsigned)((count + 7) / 8), 256, 0, st>>>((const double2*)w, (const double2*)t, n, pairs,
                                                                     count, (double2*)out);
    return cudaGetLastError();
}
cudaError_t launch_gather_cols(const void* src, int n, const int* perm, void* dst, cudaStream_t st) {
    gather_cols_kernel<<<dim3((unsigned)((n + 127) / 128), (unsigned)n), 128, 0, st>>>((const double2*)src, n, perm,
                                                                                        (double2*)dst);
    return cudaGetLastError();
}
cudaError_t launch_eig_residual(const void* fw, const void* w, const double* theta, const void* f, int n,
                                double* part, double* out2, cudaStream_t st) {
    eig_residual_kernel<<<kSpRedBlocks, kSpRedThreads, 0, st>>>((const double2*)fw, (const double2*)w, theta,
                                                               (const double2*)f, n, part);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    sum_parts_kernel<<<1, kSpRedThreads, 0, st>>>(part, 2, 1.0, 1.0, out2);
    return cudaGetLastError();
}
cudaError_t launch_spec_scale(const void* v, const double* theta, const double* alphas, int na, int which, int n,
                              void* w, cudaStream_t st) {
    const int64_t count = (int64_t)n * n;
    int gx = (int)std::min<int64_t>((count + 255) / 256, 4 * FGFRFT_SMS);
    spec_scale_kernel<<<dim3((unsigned)gx, (unsigned)na), 256, 0, st>>>((const double2*)v, theta, alphas, na, which,
                                                                        n, (double2*)w);
    return cudaGetLastError();
}
cudaError_t launch_cdiff_sq(const void* y, bool real_y, const void* t, int64_t count, void* b, double* part,
                            cudaStream_t st) {
    if (real_y)
        cdiff_sq_kernel<true><<<kSpRedBlocks, kSpRedThreads, 0, st>>>(y, (const double2*)t, count, (double2*)b, part);
    else
        cdiff_sq_kernel<false><<<kSpRedBlocks, kSpRedThreads, 0, st>>>(y, (const double2*)t, count, (double2*)b, part);
    return cudaGetLastError();
}
cudaError_t launch_cre_dot(const void* m, const void* d, bool real_d, int64_t count, double* part, cudaStream_t st) {
    if (real_d)
        cre_dot_kernel<true><<<kSpRedBlocks, kSpRedThreads, 0, st>>>((const double2*)m, d, count, part);
    else
        cre_dot_kernel<false><<<kSpRedBlocks, kSpRedThreads, 0, st>>>((const double2*)m, d, count, part);
    return cudaGetLastError();
}
cudaError_t launch_rdot(const double* a, const double* b, int64_t count, double* part, cudaStream_t st) {
    rdot_kernel<<<kSpRedBlocks, kSpRedThreads, 0, st>>>(a, b, count, part);
    return cudaGetLastError();
}
cudaError_t launch_sum_parts(const double* part, int groups, double s0, double s1, double* out, cudaStream_t st) {
    sum_parts_kernel<<<1, kSpRedThreads, 0, st>>>(part, groups, s0, s1, out);
    return cudaGetLastError();
}

}  // namespace fgb
