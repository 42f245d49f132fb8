/*
 * fgfrft_oracle.c -- CPU restatement of the FGFRFT hot path (TEST INFRASTRUCTURE).
 *
 * This file is the CHECKER, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it. The product path
 * (paper_2602_20870_b200/, libfgfrft_b200.so) never links or calls it.
 *
 * It restates, in plain C99, the scalar and elementwise parts of the reference:
 *   - sinc / sinc_deriv / sinc_coeffs  <- proj/include/fgfrft/sinc.hpp:15-63
 *   - fnv1a64 (content fingerprint)     <- proj/include/fgfrft/rng.hpp:59-67, gft.hpp:46-48
 *   - series synthesis Q = c0 I + sum_k (a_k P_k + b_k P_k^H), zero-init, diagonal,
 *     ascending k, 96x96 blocks with the transposed block read as an adjoint
 *                                        <- proj/include/fgfrft/transform.hpp:21-34, 111-136
 *   - the per-power reduction s_k = Re<M, P_k> used for dL/dalpha
 *                                        <- proj/include/fgfrft/learn.hpp:88-94 (definition)
 * Dense GEMMs (cache recursion transform.hpp:58, apply transform.hpp:140/147) are done in
 * oracle/fgfrft_oracle.py with numpy (OpenBLAS zgemm standing in for the absent Eigen GEMM).
 *
 * Storage convention (same as Eigen::MatrixXcd): column-major, interleaved (re, im) doubles;
 * element (i, j) of an n x n matrix lives at doubles [2*(i + j*n)], [2*(i + j*n) + 1].
 *
 * Arithmetic note: the pair update q += a*p + b*conj(p^T) is evaluated as
 *   t = (a*p_re) + (b*pt_re);  q_re = q_re + t      (likewise im with -b*pt_im)
 * with no fused multiply-add (build with -ffp-contract=off), the order Eigen's
 * expression template evaluates it in. Integer orders therefore give exact Kronecker
 * results and Q(-alpha) = Q(alpha)^H holds bit-for-bit.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* sinc.hpp:15-22 */
double oracle_sinc(double x) {
    if (x == nearbyint(x)) return x == 0.0 ? 1.0 : 0.0;
    if (fabs(x) < 1e-6) {
        const double px = M_PI * x;
        return 1.0 - px * px / 6.0;
    }
    return sin(M_PI * x) / (M_PI * x);
}

/* sinc.hpp:24-36 */
double oracle_sinc_deriv(double x) {
    if (x == nearbyint(x)) {
        if (x == 0.0) return 0.0;
        const long long k = (long long)x;
        return (k % 2 == 0 ? 1.0 : -1.0) / x;
    }
    if (fabs(x) < 1e-6) {
        const double pi2 = M_PI * M_PI;
        return -pi2 * x / 3.0 + pi2 * pi2 * x * x * x / 30.0;
    }
    const double px = M_PI * x;
    return cos(px) / x - sin(px) / (M_PI * x * x);
}

/* sinc.hpp:50-63; entry [n + l] holds term n. Returns -1 for l < 1 (parameter_error). */
int oracle_sinc_coeffs(double alpha, int l, double* c, double* dc) {
    if (l < 1) return -1;
    for (int n = -l; n <= l; ++n) {
        const double x = alpha - (double)n;
        if (c) c[n + l] = oracle_sinc(x);
        if (dc) dc[n + l] = oracle_sinc_deriv(x);
    }
    return 0;
}

/* rng.hpp:59-67 */
uint64_t oracle_fnv1a64(const void* data, size_t nbytes, uint64_t h) {
    const unsigned char* p = (const unsigned char*)data;
    for (size_t i = 0; i < nbytes; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

/*
 * transform.hpp:21-34 (add_scaled_pair): q += a*p + b*p^H over 96x96 blocks.
 * Column blocks j0 are independent, so they may be split over threads without
 * changing a single bit of the result.
 */
static void add_scaled_pair(double* q, double a, double b, const double* p, int64_t n, int nthreads) {
    const int64_t kb = 96;
    const int64_t nblk = (n + kb - 1) / kb;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(nthreads) if (nthreads > 1)
#endif
    for (int64_t jb = 0; jb < nblk; ++jb) {
        const int64_t j0 = jb * kb;
        const int64_t bj = (n - j0) < kb ? (n - j0) : kb;
        for (int64_t i0 = 0; i0 < n; i0 += kb) {
            const int64_t bi = (n - i0) < kb ? (n - i0) : kb;
            for (int64_t jj = 0; jj < bj; ++jj) {
                const int64_t j = j0 + jj;
                for (int64_t ii = 0; ii < bi; ++ii) {
                    const int64_t i = i0 + ii;
                    const double* pij = p + 2 * (i + j * n);
                    const double* pji = p + 2 * (j + i * n);
                    double* qij = q + 2 * (i + j * n);
                    const double tr = a * pij[0] + b * pji[0];
                    const double ti = a * pij[1] + b * (-pji[1]);
                    qij[0] = qij[0] + tr;
                    qij[1] = qij[1] + ti;
                }
            }
        }
    }
    (void)nthreads;
}

/*
 * transform.hpp:111-123 / 127-136. coef has 2l+1 entries ([n + l] = term n, i.e. the
 * SincCoeffs layout). powers: l slabs, slab k-1 holds F^k. q: n x n output.
 */
void oracle_synthesize(const double* powers, int64_t n, int l, const double* coef, double* q, int nthreads) {
    const size_t slab = (size_t)2 * (size_t)n * (size_t)n;
    memset(q, 0, slab * sizeof(double));
    for (int64_t i = 0; i < n; ++i) q[2 * (i + i * n)] = coef[l];
    for (int k = 1; k <= l; ++k)
        add_scaled_pair(q, coef[l + k], coef[l - k], powers + (size_t)(k - 1) * slab, n, nthreads);
}

/*
 * s_k = Re sum_ij conj(M_ij) (P_k)_ij for k = 1..l and s_{-k} = Re sum_ij conj(M_ij) conj((P_k)_ji)
 * with s_0 = Re tr(M) ... where M = G X^H. Then Re<G, F^k X> = s_k, so
 * dL/dalpha = sum_k c'_k s_k (learn.hpp:88-92 with dQ = sum_k c'_k F^k).
 * out has 2l+1 entries in the SincCoeffs layout. Summation: column-major order, one
 * accumulator per k (the reference never forms this sum; only its value is pinned).
 */
void oracle_power_dots(const double* powers, int64_t n, int l, const double* m, double* out) {
    const size_t slab = (size_t)2 * (size_t)n * (size_t)n;
    double s0 = 0.0;
    for (int64_t i = 0; i < n; ++i) s0 += m[2 * (i + i * n)];
    out[l] = s0;
    for (int k = 1; k <= l; ++k) {
        const double* p = powers + (size_t)(k - 1) * slab;
        double sp = 0.0, sm = 0.0;
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) {
                const double* mij = m + 2 * (i + j * n);
                const double* pij = p + 2 * (i + j * n);
                const double* pji = p + 2 * (j + i * n);
                /* Re(conj(m) * p) = m_re p_re + m_im p_im */
                sp += mij[0] * pij[0] + mij[1] * pij[1];
                /* Re(conj(m) * conj(p_ji)) = m_re p_ji_re - m_im p_ji_im */
                sm += mij[0] * pji[0] - mij[1] * pji[1];
            }
        out[l + k] = sp;
        out[l - k] = sm;
    }
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
