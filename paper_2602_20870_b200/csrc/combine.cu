// combine.cu -- the power-product route of an order sweep (real F).
//
// For A orders over one signal batch, F^a X = sum_{k=-L..L} c_k(a) F^k X (transform.hpp:111-123
// applied to X, reassociated). Once the 2L power products Z_k = F^k X are formed by ONE
// INT8-tensor-core GEMM over the stacked cache (ozgemm.cu), every order costs only a
// (2L+1)-term combination, and the MSE step needs, per order a:
//   Y_a = sum_q c_aq Z_q               (q = k + L; Z_0 = X)
//   R_a = Y_a - Xc,  loss_a = |R_a|^2 / (N B),  G_a = 2 R_a / (N B)
//   s_aq = Re<G_a, Z_q>               (the dL/dalpha contraction of learn.hpp:88-94 / 328-337)
// All of it is real arithmetic over the flat (re, im) positions p of an N x B block, so per chunk
// of 64 positions a CTA does two small DMMA GEMMs (Y = C Z_chunk, then S += G Z_chunk^T) with the
// coefficient table and the chunk in shared memory; Z is read from HBM exactly once per 64
// orders. Per-CTA partials of s and of the loss are summed in a fixed order by a second kernel
// (deterministic).
#include "common.cuh"

namespace fgb {

constexpr int kCbA = 64;    // orders per launch (rows of Y, S)
constexpr int kCbP = 64;    // positions per chunk
constexpr int kCbLdP = 68;  // doubles per staged row of 64 positions (= 4 mod 16: conflict free)
constexpr int kCbMaxT = 136;  // padded terms (2L + 1 <= 129 -> L <= 64), multiple of 8

__host__ __device__ constexpr int cb_ldc(int tp) { return tp + ((4 - tp % 16) + 16) % 16; }  // = 4 mod 16

size_t combine_smem_bytes(int tp) {
    return ((size_t)kCbA * cb_ldc(tp) + 2 * (size_t)tp * kCbLdP + 2 * kCbP) * sizeof(double);
}

int combine_max_terms() { return kCbMaxT; }

// z: 2L blocks of `count` doubles: block j < L holds F^(j+1) X, block L + j holds F^-(j+1) X.
// Warp w owns orders 8w..8w+7 for both GEMMs, so G never leaves the warp: the Y accumulators
// are turned into the A fragments of S += G Z^T with quad shuffles. The chunk ring is double
// buffered (cp.async prefetch of chunk i+1 while chunk i is multiplied): one barrier per chunk.
// MODE 0: MSE step (Y, loss, S; Y stored when y != null). MODE 1: apply (Y only, stored).
// MODE 2: dots (S += G Z^T for a caller's G = `xc`, A blocks of `count`; no Y).
// MODE 3: MSE step for a verified-orthogonal F: Y and the loss as in MODE 0, but instead of the
//   S GEMM the 2L+1 products R_q = <Xc, Z_q> and the Gram sequence gamma(d) = <X, F^d X>,
//   d = 0..2L, are accumulated (258 dot products per chunk on the FP64 pipe); S follows from
//   <Y_a, Z_q> = sum_q' c_aq' <Z_q', Z_q> = sum_q' c_aq' gamma(|q - q'|) (F^T F = I).
template <int MODE>
__global__ void __launch_bounds__(256, 1)
combine_kernel(const double* __restrict__ z, const double* __restrict__ x, const double* __restrict__ xc,
               int64_t count, int l, int tp, const double* __restrict__ coef, int n_alpha, double g_scale,
               double* __restrict__ y, double* __restrict__ spart, double* __restrict__ lpart) {
    constexpr bool kY = MODE != 2, kS = MODE != 1 && MODE != 3, kMse = MODE == 0 || MODE == 3;
    extern __shared__ __align__(16) double sm[];
    const int ldc = cb_ldc(tp);
    double* cf = sm;                       // [64][ldc]      coefficients c_aq (zero padded)
    double* zb = cf + kCbA * ldc;          // 2 x [tp][68]   chunk of every term
    double* xb = zb + 2 * tp * kCbLdP;     // 2 x [64]       Xc chunk
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    const int T = 2 * l + 1;

    for (int idx = tid; idx < kCbA * ldc; idx += 256) {
        const int a = idx / ldc, q = idx - a * ldc;
        cf[idx] = (coef && a < n_alpha && q < T) ? coef[(int64_t)a * T + q] : 0.0;
    }
    for (int idx = tid; idx < (tp - T) * kCbLdP; idx += 256) {
        zb[T * kCbLdP + idx] = 0.0;
        zb[(tp + T) * kCbLdP + idx] = 0.0;
    }

    const int64_t nchunks = (count + kCbP - 1) / kCbP;
    auto stage = [&](int64_t ch, int buf) {
        const int64_t p0 = ch * kCbP;
        const int pv = (int)((count - p0) < kCbP ? (count - p0) : kCbP);
        double* zc = zb + buf * tp * kCbLdP;
        for (int idx = tid; idx < T * (kCbP / 2); idx += 256) {
            const int q = idx / (kCbP / 2), c2 = idx - q * (kCbP / 2);
            const double* src;
            if (q == l) src = x;
            else if (q > l) src = z + (int64_t)(q - l - 1) * count;
            else src = z + (int64_t)(l + (l - q) - 1) * count;
            const bool v = 2 * c2 < pv;
            cp_async16(zc + q * kCbLdP + 2 * c2, src + p0 + (v ? 2 * c2 : 0), v);
        }
        if (kMse && tid < kCbP / 2)
            cp_async16(xb + buf * kCbP + 2 * tid, xc + p0 + (2 * tid < pv ? 2 * tid : 0), 2 * tid < pv);
    };

    double sacc[kCbMaxT / 8][2];
    const int nqb = tp / 8;
#pragma unroll
    for (int qb = 0; qb < kCbMaxT / 8; ++qb) sacc[qb][0] = sacc[qb][1] = 0.0;
    double lacc = 0.0;  // sum of R^2 over this thread's (order g of warp, positions)
    double dacc[2] = {0.0, 0.0};  // MODE 3: dot products tid and tid + 256 of the 2 (2L + 1) list
    const int a = 8 * warp + g;
    const bool a_ok = a < n_alpha;
    const double* crow = cf + a * ldc;

    int buf = 0;
    if (blockIdx.x < nchunks) stage(blockIdx.x, 0);
    cp_async_commit();
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x, buf ^= 1) {
        const int64_t p0 = ch * kCbP;
        const int pv = (int)((count - p0) < kCbP ? (count - p0) : kCbP);
        cp_async_wait<0>();
        __syncthreads();  // chunk `buf` landed for everyone; everyone is done with buffer buf^1
        if (ch + gridDim.x < nchunks) stage(ch + gridDim.x, buf ^ 1);
        cp_async_commit();
        const double* zc = zb + buf * tp * kCbLdP;
        const double* xs = xb + buf * kCbP;

        // Y (orders 8w..8w+7) x (64 positions) = C Z_chunk
        double yacc[8][2];
#pragma unroll
        for (int pb = 0; pb < 8; ++pb) yacc[pb][0] = yacc[pb][1] = 0.0;
        if (kY) {
            for (int q0 = 0; q0 < tp; q0 += 4) {
                const double av = crow[q0 + t];
                const double* zrow = zc + (q0 + t) * kCbLdP + g;
#pragma unroll
                for (int pb = 0; pb < 8; ++pb) dmma884(yacc[pb][0], yacc[pb][1], av, zrow[8 * pb]);
            }
        }
        if (MODE == 3) {
            // R_q = <Xc, Z_q> (j < T) and gamma(d) (j = T + d): rows (L, L + d) for d <= L, else
            // (0, d). Position order rotated by j: the 32 lanes read 32 rows without bank conflicts.
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = tid + 256 * h;
                if (j < 2 * T) {
                    const double *u, *v;
                    if (j < T) {
                        u = xs;
                        v = zc + j * kCbLdP;
                    } else {
                        const int d = j - T;
                        u = zc + (d <= l ? l : 0) * kCbLdP;
                        v = zc + (d <= l ? l + d : d) * kCbLdP;
                    }
                    double acc = 0.0;
#pragma unroll 8
                    for (int i = 0; i < kCbP; ++i) {
                        const int p = (i + j) & (kCbP - 1);
                        acc = fma(u[p], v[p], acc);
                    }
                    dacc[h] += acc;
                }
            }
        }
        if (kMse) {
            // residual, loss, G (in place of Y), optional Y store
#pragma unroll
            for (int pb = 0; pb < 8; ++pb) {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int p = 8 * pb + 2 * t + e;
                    const bool ok = p < pv && a_ok;
                    if (y && ok) y[(int64_t)a * count + p0 + p] = yacc[pb][e];
                    const double r = ok ? yacc[pb][e] - xs[p] : 0.0;
                    lacc += r * r;
                    yacc[pb][e] = r * g_scale;
                }
            }
        } else if (MODE == 1) {
#pragma unroll
            for (int pb = 0; pb < 8; ++pb)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int p = 8 * pb + 2 * t + e;
                    if (p < pv && a_ok) y[(int64_t)a * count + p0 + p] = yacc[pb][e];
                }
            continue;
        } else {
            // the caller's G, loaded in the accumulator layout (rows a, positions 8pb + 2t + e)
#pragma unroll
            for (int pb = 0; pb < 8; ++pb)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int p = 8 * pb + 2 * t + e;
                    yacc[pb][e] = (p < pv && a_ok) ? xc[(int64_t)a * count + p0 + p] : 0.0;
                }
        }
        if (MODE == 3) continue;
        // S (orders 8w..8w+7) x (terms) += G_chunk Z_chunk^T. A fragment of k-step (pb, h):
        // lane (g, t) needs G[g][8pb + 4h + t], held by lane (g, 2h + (t >> 1)) as element t & 1.
#pragma unroll
        for (int pb = 0; pb < 8; ++pb) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int src = (lane & ~3) | (2 * h + (t >> 1));
                const double v0 = __shfl_sync(0xffffffffu, yacc[pb][0], src);
                const double v1 = __shfl_sync(0xffffffffu, yacc[pb][1], src);
                const double av = (t & 1) ? v1 : v0;
                const double* zcol = zc + g * kCbLdP + 8 * pb + 4 * h + t;
#pragma unroll
                for (int qb = 0; qb < kCbMaxT / 8; ++qb)
                    if (qb < nqb) dmma884(sacc[qb][0], sacc[qb][1], av, zcol[8 * qb * kCbLdP]);
            }
        }
    }
    cp_async_wait<0>();
    if (MODE == 3) {
        double* dp = spart + (int64_t)blockIdx.x * 2 * T;  // [cta][R_0..R_2L, gamma_0..gamma_2L]
#pragma unroll
        for (int h = 0; h < 2; ++h)
            if (tid + 256 * h < 2 * T) dp[tid + 256 * h] = dacc[h];
        lacc += __shfl_xor_sync(0xffffffffu, lacc, 1);
        lacc += __shfl_xor_sync(0xffffffffu, lacc, 2);
        if (t == 0) lpart[(int64_t)blockIdx.x * kCbA + a] = lacc;
        return;
    }
    if (!kS) return;
    // partials: spart[cta][a][q] (q < tp), lpart[cta][a]
    double* sp = spart + (int64_t)blockIdx.x * kCbA * tp;
#pragma unroll
    for (int qb = 0; qb < kCbMaxT / 8; ++qb)
        if (qb < nqb) {
            sp[a * tp + 8 * qb + 2 * t] = sacc[qb][0];
            sp[a * tp + 8 * qb + 2 * t + 1] = sacc[qb][1];
        }
    lacc += __shfl_xor_sync(0xffffffffu, lacc, 1);
    lacc += __shfl_xor_sync(0xffffffffu, lacc, 2);
    if (t == 0) lpart[(int64_t)blockIdx.x * kCbA + a] = lacc;
}

// ---------------------------------------------------------------------------------------------
// Y-only forms for an orthogonal F (MODE 3) and for apply (MODE 1), two CTAs per SM:
// the coefficient fragments live in registers (34 per lane), the chunk ring holds 32 positions of
// every term (2 x 39 KB), and the three Gram/residual rows <X, Z_q>, <Z_-L, Z_q>, <Xc, Z_q> are
// one extra DMMA GEMV per chunk (rows of the A fragment: X, Z_-L, Xc).
constexpr int kCyP = 32;    // positions per chunk
constexpr int kCyLd = 36;   // doubles per staged row (= 4 mod 16)

size_t combine_y_smem_bytes(int tp) { return (2 * (size_t)tp * kCyLd + 2 * kCyP) * sizeof(double); }

template <bool GRAM>
__global__ void __launch_bounds__(256, 2)
combine_y_kernel(const double* __restrict__ z, const double* __restrict__ x, const double* __restrict__ xc,
                 int64_t count, int l, int tp, const double* __restrict__ coef, int n_alpha, double* __restrict__ y,
                 double* __restrict__ dpart, double* __restrict__ lpart) {
    extern __shared__ __align__(16) double sm[];
    double* zb = sm;                       // 2 x [tp][36]
    double* xb = zb + 2 * tp * kCyLd;      // 2 x [32]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    const int T = 2 * l + 1;
    const int a = 8 * warp + g;
    const bool a_ok = a < n_alpha;
    const int nks = tp / 4;

    double creg[kCbMaxT / 4];
#pragma unroll
    for (int k = 0; k < kCbMaxT / 4; ++k) {
        const int q = 4 * k + t;
        creg[k] = (a_ok && q < T) ? coef[(int64_t)a * T + q] : 0.0;
    }
    for (int idx = tid; idx < (tp - T) * kCyLd; idx += 256) {
        zb[T * kCyLd + idx] = 0.0;
        zb[(tp + T) * kCyLd + idx] = 0.0;
    }

    const int64_t nchunks = (count + kCyP - 1) / kCyP;
    auto stage = [&](int64_t ch, int buf) {
        const int64_t p0 = ch * kCyP;
        const int pv = (int)((count - p0) < kCyP ? (count - p0) : kCyP);
        double* zc = zb + buf * tp * kCyLd;
        for (int idx = tid; idx < T * (kCyP / 2); idx += 256) {
            const int q = idx / (kCyP / 2), c2 = idx - q * (kCyP / 2);
            const double* src;
            if (q == l) src = x;
            else if (q > l) src = z + (int64_t)(q - l - 1) * count;
            else src = z + (int64_t)(l + (l - q) - 1) * count;
            const bool v = 2 * c2 < pv;
            cp_async16(zc + q * kCyLd + 2 * c2, src + p0 + (v ? 2 * c2 : 0), v);
        }
        if (GRAM && tid < kCyP / 2)
            cp_async16(xb + buf * kCyP + 2 * tid, xc + p0 + (2 * tid < pv ? 2 * tid : 0), 2 * tid < pv);
    };

    double lacc = 0.0;
    double dacc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};  // q-blocks warp, warp + 8, warp + 16
    int buf = 0;
    if (blockIdx.x < nchunks) stage(blockIdx.x, 0);
    cp_async_commit();
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x, buf ^= 1) {
        const int64_t p0 = ch * kCyP;
        const int pv = (int)((count - p0) < kCyP ? (count - p0) : kCyP);
        cp_async_wait<0>();
        __syncthreads();
        if (ch + gridDim.x < nchunks) stage(ch + gridDim.x, buf ^ 1);
        cp_async_commit();
        const double* zc = zb + buf * tp * kCyLd;
        const double* xs = xb + buf * kCyP;

        double yacc[4][2];
#pragma unroll
        for (int pb = 0; pb < 4; ++pb) yacc[pb][0] = yacc[pb][1] = 0.0;
#pragma unroll
        for (int k = 0; k < kCbMaxT / 4; ++k) {
            if (k < nks) {
                const double* zrow = zc + (4 * k + t) * kCyLd + g;
#pragma unroll
                for (int pb = 0; pb < 4; ++pb) dmma884(yacc[pb][0], yacc[pb][1], creg[k], zrow[8 * pb]);
            }
        }
#pragma unroll
        for (int pb = 0; pb < 4; ++pb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int p = 8 * pb + 2 * t + e;
                const bool ok = p < pv && a_ok;
                if (y && ok) y[(int64_t)a * count + p0 + p] = yacc[pb][e];
                if (GRAM) {
                    const double r = ok ? yacc[pb][e] - xs[p] : 0.0;
                    lacc += r * r;
                }
            }
        if (GRAM) {
            // rows: g = 0 -> X (term L), g = 1 -> Z_-L (term 0), g = 2 -> Xc, else 0
#pragma unroll
            for (int p4 = 0; p4 < kCyP; p4 += 4) {
                const double av = g == 0 ? zc[l * kCyLd + p4 + t] : g == 1 ? zc[p4 + t] : g == 2 ? xs[p4 + t] : 0.0;
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    const int qb = warp + 8 * r;
                    if (8 * qb < tp) dmma884(dacc[r][0], dacc[r][1], av, zc[(8 * qb + g) * kCyLd + p4 + t]);
                }
            }
        }
    }
    cp_async_wait<0>();
    if (!GRAM) return;
    // partials: dpart[cta][row 0..2][tp], lpart[cta][a]
    double* dp = dpart + (int64_t)blockIdx.x * 3 * tp;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const int qb = warp + 8 * r;
        if (8 * qb < tp && g < 3) {
            dp[g * tp + 8 * qb + 2 * t] = dacc[r][0];
            dp[g * tp + 8 * qb + 2 * t + 1] = dacc[r][1];
        }
    }
    lacc += __shfl_xor_sync(0xffffffffu, lacc, 1);
    lacc += __shfl_xor_sync(0xffffffffu, lacc, 2);
    if (t == 0) lpart[(int64_t)blockIdx.x * kCbA + a] = lacc;
}

// rg[0..T) = R_q = <Xc, Z_q>, rg[T + d] = gamma(d): <X, Z_d> (row 0, q = L + d) for d <= L,
// <Z_-L, Z_(d-L)> (row 1, q = d) for d > L. loss as in combine_reduce_kernel.
__global__ void gram3_reduce_kernel(const double* __restrict__ dpart, const double* __restrict__ lpart, int ctas,
                                    int tp, int l, int n_alpha, double norm, double* __restrict__ rg,
                                    double* __restrict__ loss) {
    const int T = 2 * l + 1;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx < 2 * T) {
        int row, col;
        if (idx < T) {
            row = 2;
            col = idx;
        } else {
            const int d = idx - T;
            row = d <= l ? 0 : 1;
            col = d <= l ? l + d : d;
        }
        double acc = 0.0;
        for (int c = 0; c < ctas; ++c) acc += dpart[((int64_t)c * 3 + row) * tp + col];
        rg[idx] = acc;
    }
    if (idx < n_alpha) {
        double acc = 0.0;
        for (int c = 0; c < ctas; ++c) acc += lpart[(int64_t)c * kCbA + idx];
        loss[idx] = acc * norm;
    }
}

// s[a][q] = sum_cta spart (fixed order), loss[a] = norm * sum_cta lpart
__global__ void combine_reduce_kernel(const double* __restrict__ spart, const double* __restrict__ lpart, int ctas,
                                      int tp, int T, int n_alpha, double norm, double* __restrict__ s,
                                      double* __restrict__ loss) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx < n_alpha * T) {
        const int a = idx / T, q = idx - a * T;
        double acc = 0.0;
        for (int c = 0; c < ctas; ++c) acc += spart[((int64_t)c * kCbA + a) * tp + q];
        s[idx] = acc;
    }
    if (loss && idx < n_alpha) {
        double acc = 0.0;
        for (int c = 0; c < ctas; ++c) acc += lpart[(int64_t)c * kCbA + idx];
        loss[idx] = acc * norm;
    }
}

// MODE 3: rg[0..2T) = sum_cta of (R, gamma) partials, loss as in combine_reduce_kernel.
__global__ void gram_reduce_kernel(const double* __restrict__ dpart, const double* __restrict__ lpart, int ctas, int T,
                                   int n_alpha, double norm, double* __restrict__ rg, double* __restrict__ loss) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx < 2 * T) {
        double acc = 0.0;
        for (int c = 0; c < ctas; ++c) acc += dpart[(int64_t)c * 2 * T + idx];
        rg[idx] = acc;
    }
    if (idx < n_alpha) {
        double acc = 0.0;
        for (int c = 0; c < ctas; ++c) acc += lpart[(int64_t)c * kCbA + idx];
        loss[idx] = acc * norm;
    }
}

// s[a][q] = g_scale * (sum_q' c_aq' gamma(|q - q'|) - R_q): one CTA per order.
__global__ void gram_s_kernel(const double* __restrict__ coef, const double* __restrict__ rg, int T, double g_scale,
                              double* __restrict__ s) {
    const int a = blockIdx.x;
    const double* c = coef + (int64_t)a * T;
    const double* gam = rg + T;
    for (int q = threadIdx.x; q < T; q += blockDim.x) {
        double acc = 0.0;
        for (int q2 = 0; q2 < T; ++q2) acc = fma(c[q2], gam[q > q2 ? q - q2 : q2 - q], acc);
        s[(int64_t)a * T + q] = g_scale * (acc - rg[q]);
    }
}

int combine_ctas() { return FGFRFT_SMS; }

// out += sum_ij (G_ij - delta_ij)^2 over an n x n column-major G (orthogonality residual of F).
__global__ void ortho_residual_kernel(const double* __restrict__ g, int n, double* out) {
    double acc = 0.0;
    const int64_t total = (int64_t)n * n;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx % n, j = idx / n;
        const double v = g[idx] - (i == j ? 1.0 : 0.0);
        acc = fma(v, v, acc);
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ double red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (threadIdx.x == 0) atomicAdd(out, acc);
    }
}

cudaError_t launch_ortho_residual(const double* g, int n, double* out, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), stream);
    if (e != cudaSuccess) return e;
    ortho_residual_kernel<<<2 * FGFRFT_SMS, 256, 0, stream>>>(g, n, out);
    return cudaGetLastError();
}

size_t combine_partial_elems(int tp) {
    const size_t a = (size_t)FGFRFT_SMS * kCbA * (tp + 1) + 4 * (size_t)tp;
    const size_t b = (size_t)2 * FGFRFT_SMS * (3 * tp + kCbA) + 4 * (size_t)tp;
    return a > b ? a : b;
}

template <int MODE>
static cudaError_t combine_attr() {
    static PerDeviceOnce done;
    return done.run([] {
        return cudaFuncSetAttribute(combine_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)combine_smem_bytes(kCbMaxT));
    });
}

// mode 0 (MSE: xc = clean signals, y optional), 1 (apply: y required), 2 (dots: xc = G, A blocks).
// n_alpha <= 64, 2l + 1 <= 136; count = 2 N B (even). partial >= combine_partial_elems doubles.
cudaError_t launch_combine(int mode, const double* z, const double* x, const double* xc, int64_t count, int l,
                           const double* coef, int n_alpha, double norm, double* y, double* partial, double* s,
                           double* loss, cudaStream_t stream) {
    const int T = 2 * l + 1, tp = (T + 7) / 8 * 8;
    if (n_alpha < 1 || n_alpha > kCbA || tp > kCbMaxT || count % 2 || mode < 0 || mode > 3) return cudaErrorInvalidValue;
    const size_t smem = combine_smem_bytes(tp);
    const int64_t nchunks = (count + kCbP - 1) / kCbP;
    const int ctas = (int)(nchunks < FGFRFT_SMS ? nchunks : FGFRFT_SMS);
    double* spart = partial;
    double* lpart = partial + (size_t)ctas * kCbA * tp;
    cudaError_t e;
    switch (mode) {
        case 0:
            if ((e = combine_attr<0>()) != cudaSuccess) return e;
            combine_kernel<0><<<ctas, 256, smem, stream>>>(z, x, xc, count, l, tp, coef, n_alpha, 2.0 * norm, y, spart,
                                                           lpart);
            break;
        case 1:
        case 3: {
            const size_t ysm = combine_y_smem_bytes(tp);
            static PerDeviceOnce yattr;
            if ((e = yattr.run([] {
                     cudaError_t r = cudaFuncSetAttribute(combine_y_kernel<true>,
                                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                          (int)combine_y_smem_bytes(kCbMaxT));
                     if (r != cudaSuccess) return r;
                     return cudaFuncSetAttribute(combine_y_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)combine_y_smem_bytes(kCbMaxT));
                 })) != cudaSuccess)
                return e;
            const int64_t ych = (count + kCyP - 1) / kCyP;
            const int yctas = (int)(ych < 2 * FGFRFT_SMS ? ych : 2 * FGFRFT_SMS);
            if (mode == 1) {
                combine_y_kernel<false><<<yctas, 256, ysm, stream>>>(z, x, xc, count, l, tp, coef, n_alpha, y, nullptr,
                                                                    nullptr);
                return cudaGetLastError();
            }
            double* dpart = partial;                                 // [yctas][3][tp]
            double* lp = partial + (size_t)yctas * 3 * tp;           // [yctas][64]
            double* rg = lp + (size_t)yctas * kCbA;                  // [2T]
            combine_y_kernel<true><<<yctas, 256, ysm, stream>>>(z, x, xc, count, l, tp, coef, n_alpha, y, dpart, lp);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
            const int threads = 256, blocks = (2 * T + threads - 1) / threads;
            gram3_reduce_kernel<<<blocks, threads, 0, stream>>>(dpart, lp, yctas, tp, l, n_alpha, norm, rg, loss);
            gram_s_kernel<<<n_alpha, 128, 0, stream>>>(coef, rg, T, 2.0 * norm, s);
            return cudaGetLastError();
        }
        default:
            if ((e = combine_attr<2>()) != cudaSuccess) return e;
            combine_kernel<2><<<ctas, 256, smem, stream>>>(z, x, xc, count, l, tp, coef, n_alpha, 0.0, y, spart,
                                                           lpart);
            break;
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int threads = 256, blocks = (n_alpha * T + threads - 1) / threads;
    combine_reduce_kernel<<<blocks, threads, 0, stream>>>(spart, lpart, ctas, tp, T, n_alpha, norm, s,
                                                          mode == 0 ? loss : nullptr);
    return cudaGetLastError();
}

}  // namespace fgb

namespace fgb {

// ---------------------------------------------------------------------------------------------
// Orthogonal-F sweep with the combination on the INT8 tensor cores (see capi.cu power route):
// per signal column j: colsq = |x_j|^2, colxc = Re<xc_j, x_j>; one CTA per column.
__global__ void __launch_bounds__(256) colstats_kernel(const double* __restrict__ x, const double* __restrict__ xc,
                                                       int n, double* __restrict__ colsq, double* __restrict__ colxc) {
    const int j = blockIdx.x;
    const double* xj = x + (int64_t)j * 2 * n;
    const double* cj = xc + (int64_t)j * 2 * n;
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < 2 * n; i += 256) {
        a = fma(xj[i], xj[i], a);
        b = fma(xj[i], cj[i], b);
    }
    __shared__ double ra[8], rb[8];
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0) {
        ra[threadIdx.x >> 5] = a;
        rb[threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sa = 0.0, sb = 0.0;
        for (int w = 0; w < 8; ++w) {
            sa += ra[w];
            sb += rb[w];
        }
        colsq[j] = sa;
        colxc[j] = sb;
    }
}

// e_j: 2^e_j > |x_j| (1 + 2^-20) >= every |(F^k X)[i, j]| for orthogonal F (the combine GEMM
// reads the row exponent of position p as e_(p / 2n)); rg[T + 0] = gamma(0) = |X|^2 and
// rg[L] = R_0 = <Xc, X> (fixed-order sums).
__global__ void expo_kernel(const double* __restrict__ colsq, const double* __restrict__ colxc, int b,
                            int* __restrict__ ecol, double* __restrict__ rg, int l) {
    for (int j = threadIdx.x; j < b; j += blockDim.x) {
        int e = 0;
        const double nrm = sqrt(colsq[j]) * (1.0 + 0x1p-20);
        if (nrm > 0.0) frexp(nrm, &e);
        ecol[j] = e;
    }
    if (threadIdx.x == 0) {
        double g0 = 0.0, r0 = 0.0;
        for (int j = 0; j < b; ++j) {
            g0 += colsq[j];
            r0 += colxc[j];
        }
        const int T = 2 * l + 1;
        rg[T] = g0;
        rg[l] = r0;
    }
}

// dlda[a] = sum_q dc[a][q] s[a][q] with s from the Gram form (gram_s_kernel fused): one CTA per order.
__global__ void gram_s_dlda_kernel(const double* __restrict__ coef, const double* __restrict__ dcoef,
                                   const double* __restrict__ rg, int T, double g_scale, double* __restrict__ s,
                                   double* __restrict__ dlda) {
    const int a = blockIdx.x;
    const double* c = coef + (int64_t)a * T;
    const double* gam = rg + T;
    __shared__ double sv[272];
    for (int q = threadIdx.x; q < T; q += blockDim.x) {
        double acc = 0.0;
        for (int q2 = 0; q2 < T; ++q2) acc = fma(c[q2], gam[q > q2 ? q - q2 : q2 - q], acc);
        const double v = g_scale * (acc - rg[q]);
        sv[q] = v;
        if (s) s[(int64_t)a * T + q] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // ascending q, as coef_dot_kernel
        const double* dc = dcoef + (int64_t)a * T;
        double acc = 0.0;
        for (int q = 0; q < T; ++q) acc += dc[q] * sv[q];
        dlda[a] = acc;
    }
}

// Gram partials [cta][4][128][3] (thread row lrow -> term kk = lrow % tp2) -> rg:
//   R_q (q = k + L): k > 0 -> <Xc, Z_k> = part1[kk = k - 1]; k < 0 -> part1[kk = L - k - 1]
//   gamma(d): 1 <= d <= L -> <X, Z_d> = part0[kk = d - 1]; L < d <= 2L -> <Z_-L, Z_(d-L)> =
//   part2[kk = d - L - 1] (F^T F = I: <F^-L X, F^k X> = <X, F^(k+L) X>)
__device__ __forceinline__ double block_sum128(double v, double* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    const double s = red[0] + red[1] + red[2] + red[3];  // fixed order
    __syncthreads();
    return s;
}

// one CTA (128 threads) per term kk; entries (cta, h, r = kk + m tp2) strided over the threads
__global__ void __launch_bounds__(128) gram_terms_kernel(const double* __restrict__ part, int ctas, int tp2, int l,
                                                         double* __restrict__ rg) {
    const int kk = blockIdx.x;
    const int per = 128 / tp2, entries = ctas * 4 * per;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int e = threadIdx.x; e < entries; e += 128) {
        const int c = e / (4 * per), rem = e - c * 4 * per, h = rem / per, m = rem - h * per;
        const double* p = part + (((int64_t)c * 4 + h) * 128 + kk + m * tp2) * 3;
        s0 += p[0];
        s1 += p[1];
        s2 += p[2];
    }
    __shared__ double red[4];
    s0 = block_sum128(s0, red);
    s1 = block_sum128(s1, red);
    s2 = block_sum128(s2, red);
    if (threadIdx.x != 0) return;
    const int T = 2 * l + 1;
    const int k = kk < l ? kk + 1 : -(kk - l + 1);
    rg[l + k] = s1;                       // R_(L+k)
    if (k > 0) {
        rg[T + k] = s0;                   // gamma(k), k = 1..L
        rg[T + l + k] = s2;               // gamma(L + k) = <Z_-L, Z_k>
    }
}

// loss[a] = norm * sum over [cta][4][4][16] partials (order a = q * 16 + c)
__global__ void __launch_bounds__(128) loss3_kernel(const double* __restrict__ part, int ctas, int n_alpha,
                                                    double norm, double* __restrict__ loss) {
    const int a = blockIdx.x;
    const int h = a >> 4, c = a & 15;
    double acc = 0.0;
    for (int e = threadIdx.x; e < ctas * 4; e += 128) {
        const int t = e >> 2, lg = e & 3;
        acc += part[(((int64_t)t * 4 + h) * 4 + lg) * 16 + c];
    }
    __shared__ double red[4];
    acc = block_sum128(acc, red);
    if (threadIdx.x == 0) loss[a] = acc * norm;
}

cudaError_t launch_colstats(const double* x, const double* xc, int n, int b, double* colsq, double* colxc, int* ecol,
                            double* rg, int l, cudaStream_t st) {
    colstats_kernel<<<b, 256, 0, st>>>(x, xc, n, colsq, colxc);
    expo_kernel<<<1, 256, 0, st>>>(colsq, colxc, b, ecol, rg, l);
    return cudaGetLastError();
}

cudaError_t launch_gram_s_dlda(const double* coef, const double* dcoef, const double* rg, int n_alpha, int l,
                               double norm, double* s, double* dlda, cudaStream_t st) {
    if (2 * l + 1 > 272) return cudaErrorInvalidValue;
    gram_s_dlda_kernel<<<n_alpha, 128, 0, st>>>(coef, dcoef, rg, 2 * l + 1, 2.0 * norm, s, dlda);
    return cudaGetLastError();
}

cudaError_t launch_gram_terms(const double* part, int ctas, int tp2, int l, double* rg, cudaStream_t st) {
    gram_terms_kernel<<<2 * l, 128, 0, st>>>(part, ctas, tp2, l, rg);
    return cudaGetLastError();
}

cudaError_t launch_loss3(const double* part, int ctas, int n_alpha, double norm, double* loss, cudaStream_t st) {
    loss3_kernel<<<n_alpha, 128, 0, st>>>(part, ctas, n_alpha, norm, loss);
    return cudaGetLastError();
}

cudaError_t launch_gram_s(const double* coef, const double* rg, int n_alpha, int l, double norm, double* s,
                          cudaStream_t st) {
    gram_s_kernel<<<n_alpha, 128, 0, st>>>(coef, rg, 2 * l + 1, 2.0 * norm, s);
    return cudaGetLastError();
}

}  // namespace fgb

namespace fgb {

// ---------------------------------------------------------------------------------------------
// Node route of an order sweep (capi.cu): the series operator is polynomial-interpolated in the
// order over r Chebyshev nodes a_j of the sweep's interval, Q(a) = sum_j l_j(a) Q(a_j) + O(1e-15),
// dQ/da(a) = sum_j l_j'(a) Q(a_j); with Z'_j = Q(a_j) X formed by one INT8 GEMM, per order a over
// the flat (re, im) positions p of the N x B block:
//   Y_a = sum_j P[a][j] Z'_j,  loss_a = |Y_a - Xc|^2 / (N B),
//   dL/da = 2/(N B) <Y_a - Xc, dY_a> = 2/(N B) sum_j P[A + a][j] ((G P[a])_j - h_j)
// with the node Gram G = Z'^T Z' (r x r) and h = Z'^T Xc: dY is never formed. Warp w owns orders
// 8w..8w+7 of Y (coefficient fragments in registers), so the residual and the loss stay in the
// accumulators' lanes; the Gram [Z'; Xc] [Z'; Xc]^T (Xc staged as row r of the chunk) is
// accumulated by upper-triangular 8x8 DMMA tiles, warp w taking positions 4w..4w+3 of every
// chunk. 32-position chunks double buffered through cp.async, two CTAs per SM. MSE = false: Y only.
constexpr int kNdMaxR = 48;
constexpr int kNdP = 64;                           // positions per chunk (one __syncthreads per chunk)
constexpr int kNdLd = 68;                          // = 4 mod 16: the DMMA fragment loads are conflict free
constexpr int kNdT = (kNdMaxR + 1 + 7) / 8;        // 8-row tiles of [Z'; Xc]
constexpr int kNdPairs = kNdT * (kNdT + 1) / 2;    // upper-triangular tile pairs of the Gram

__host__ __device__ inline int node_rows8(int r) { return (r + 1 + 7) / 8 * 8; }
size_t node_smem_bytes(int r) { return 2 * (size_t)node_rows8(r) * kNdLd * sizeof(double); }
int node_max_terms() { return kNdMaxR; }

template <bool MSE, int T>  // T = node_rows8(r) / 8
__global__ void __launch_bounds__(256, 2)
node_combine_kernel(const double* __restrict__ zin, const double* __restrict__ xc, int64_t count, int r, int rp,
                    const double* __restrict__ pc, int n_alpha, double* __restrict__ y, double* __restrict__ lpart,
                    double* __restrict__ gpart) {
    extern __shared__ __align__(16) double sm[];
    constexpr int r8 = 8 * T, t8 = T;
    double* zb = sm;  // 2 x [r8][36]: rows 0..r-1 Z', row r Xc, the rest zero
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    const int a = 8 * warp + g;
    const bool a_ok = a < n_alpha;
    const int nks = rp / 4;
    double cy[2 * T];
#pragma unroll
    for (int k = 0; k < 2 * T; ++k) {
        const int q = 4 * k + t;
        cy[k] = (a_ok && q < r) ? pc[(int64_t)a * rp + q] : 0.0;
    }
    const int zrow0 = MSE ? r + 1 : r;
    for (int idx = tid; idx < (r8 - zrow0) * kNdLd; idx += 256) {  // padded rows stay zero
        zb[zrow0 * kNdLd + idx] = 0.0;
        zb[(r8 + zrow0) * kNdLd + idx] = 0.0;
    }
    const int64_t nchunks = (count + kNdP - 1) / kNdP;
    auto stage = [&](int64_t ch, int buf) {
        const int64_t p0 = ch * kNdP;
        const int pv = (int)((count - p0) < kNdP ? (count - p0) : kNdP);
        double* zc = zb + buf * r8 * kNdLd;
        for (int idx = tid; idx < r * (kNdP / 2); idx += 256) {
            const int q = idx / (kNdP / 2), c2 = idx - q * (kNdP / 2);
            const bool v = 2 * c2 < pv;
            cp_async16(zc + q * kNdLd + 2 * c2, zin + (int64_t)q * count + p0 + (v ? 2 * c2 : 0), v);
        }
        if (MSE && tid < kNdP / 2)
            cp_async16(zc + r * kNdLd + 2 * tid, xc + p0 + (2 * tid < pv ? 2 * tid : 0), 2 * tid < pv);
    };
    double lacc = 0.0;
    double gacc[T * (T + 1) / 2][2];
#pragma unroll
    for (int i = 0; i < T * (T + 1) / 2; ++i) gacc[i][0] = gacc[i][1] = 0.0;
    int buf = 0;
    if (blockIdx.x < nchunks) stage(blockIdx.x, 0);
    cp_async_commit();
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x, buf ^= 1) {
        const int64_t p0 = ch * kNdP;
        const int pv = (int)((count - p0) < kNdP ? (count - p0) : kNdP);
        cp_async_wait<0>();
        __syncthreads();
        if (ch + gridDim.x < nchunks) stage(ch + gridDim.x, buf ^ 1);
        cp_async_commit();
        const double* zc = zb + buf * r8 * kNdLd;
        const double* xs = zc + r * kNdLd;
        constexpr int PB = kNdP / 8;  // 8-position blocks per chunk
        double yacc[PB][2];
#pragma unroll
        for (int pb = 0; pb < PB; ++pb) yacc[pb][0] = yacc[pb][1] = 0.0;
#pragma unroll
        for (int k = 0; k < 2 * T; ++k) {
            if (k < nks) {
                const double* zrow = zc + (4 * k + t) * kNdLd + g;
#pragma unroll
                for (int pb = 0; pb < PB; ++pb) dmma884(yacc[pb][0], yacc[pb][1], cy[k], zrow[8 * pb]);
            }
        }
        if (MSE) {
#pragma unroll
            for (int cg = 0; cg < kNdP / 32; ++cg) {  // K = 4 positions per warp per 32-position group
                const int col = 32 * cg + 4 * warp + t;
                int pi = 0;
#pragma unroll
                for (int mt = 0; mt < T; ++mt) {
                    const double av = mt < t8 ? zc[(8 * mt + g) * kNdLd + col] : 0.0;
#pragma unroll
                    for (int nt = mt; nt < T; ++nt, ++pi)
                        if (nt < t8) dmma884(gacc[pi][0], gacc[pi][1], av, zc[(8 * nt + g) * kNdLd + col]);
                }
            }
        }
#pragma unroll
        for (int pb = 0; pb < PB; ++pb)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int p = 8 * pb + 2 * t + e;
                const bool ok = p < pv && a_ok;
                if (y && ok) y[(int64_t)a * count + p0 + p] = yacc[pb][e];
                if (MSE) {
                    const double res = ok ? yacc[pb][e] - xs[p] : 0.0;
                    lacc = fma(res, res, lacc);
                }
            }
    }
    cp_async_wait<0>();
    if (!MSE) return;
    lacc += __shfl_xor_sync(0xffffffffu, lacc, 1);
    lacc += __shfl_xor_sync(0xffffffffu, lacc, 2);
    if (t == 0) lpart[(int64_t)blockIdx.x * kCbA + a] = lacc;
    // the 8 warps' Gram tiles summed in warp order through shared memory (deterministic)
    const int npairs = t8 * (t8 + 1) / 2;
    __syncthreads();
    double* gs = zb;  // npairs x 64 <= 2 r8 kNdLd
    for (int w = 0; w < 8; ++w) {
        if (warp == w) {
            int pi = 0, pc2 = 0;
#pragma unroll
            for (int mt = 0; mt < T; ++mt)
#pragma unroll
                for (int nt = mt; nt < T; ++nt, ++pi)
                    if (nt < t8 && mt < t8) {
                        pc2 = (mt * (2 * t8 - mt + 1)) / 2 + (nt - mt);  // compact pair index
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            double* d = gs + pc2 * 64 + g * 8 + 2 * t + e;
                            *d = (w == 0 ? 0.0 : *d) + gacc[pi][e];
                        }
                    }
        }
        __syncthreads();
    }
    for (int idx = tid; idx < npairs * 64; idx += 256) gpart[(int64_t)blockIdx.x * kNdPairs * 64 + idx] = gs[idx];
}

// G = sum over CTAs of the Gram partials (fixed order): a block per 32 tile elements, lane =
// element (coalesced), warp w sums the CTAs c = w mod 16 (independent loads), then a fixed-order
// sum over the 16 warps -- the serial per-element chain over ~300 partials was latency-bound.
__global__ void __launch_bounds__(512) node_gram_reduce_kernel(const double* __restrict__ gpart, int ctas, int elems,
                                                               double* __restrict__ gsum) {
    __shared__ double red[16][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, i = blockIdx.x * 32 + lane;
    double s = 0.0;
    if (i < elems) {
#pragma unroll 4
        for (int c = w; c < ctas; c += 16) s += gpart[(int64_t)c * kNdPairs * 64 + i];
    }
    red[w][lane] = s;
    __syncthreads();
    if (w == 0 && i < elems) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q) t += red[q][lane];
        gsum[i] = t;
    }
}

// one CTA per order: loss from the per-CTA partials (fixed-order tree), dL/da from the Gram
__global__ void __launch_bounds__(128) node_reduce_kernel(const double* __restrict__ lpart,
                                                          const double* __restrict__ gsum, int ctas, int r, int rp,
                                                          const double* __restrict__ pc, int n_alpha, double norm,
                                                          double* __restrict__ loss, double* __restrict__ dlda) {
    __shared__ double sl[4], sv[kNdMaxR + 1];
    const int a = blockIdx.x, t = threadIdx.x;
    const int t8 = node_rows8(r) / 8;
    auto gval = [&](int i, int j) {  // G[i][j] from the compact upper-triangular tiles
        if (i / 8 > j / 8) {
            const int s = i;
            i = j;
            j = s;
        }
        const int mt = i / 8, nt = j / 8, pcx = (mt * (2 * t8 - mt + 1)) / 2 + (nt - mt);
        return gsum[pcx * 64 + (i & 7) * 8 + (j & 7)];
    };
    double l = 0.0;
    for (int c = t; c < ctas; c += 128) l += lpart[(int64_t)c * kCbA + a];
    for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if ((t & 31) == 0) sl[t >> 5] = l;
    if (t < r) {  // v_j = (G P[a])_j - h_j = <Z'_j, Y_a - Xc>
        double v = -gval(t, r);
        for (int k = 0; k < r; ++k) v = fma(pc[(int64_t)a * rp + k], gval(t, k), v);
        sv[t] = v;
    }
    __syncthreads();
    if (t == 0) {
        double d = 0.0;
        for (int j = 0; j < r; ++j) d = fma(pc[(int64_t)(n_alpha + a) * rp + j], sv[j], d);
        loss[a] = norm * ((sl[0] + sl[1]) + (sl[2] + sl[3]));
        dlda[a] = 2.0 * norm * d;
    }
}

// W_j[i, i] += d[j] for r row-stacked n x n operators (the identity term of the series)
__global__ void add_diag_kernel(double* __restrict__ w, int n, int64_t stride, const double* __restrict__ d, int r) {
    const int j = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && j < r) w[(int64_t)j * stride + (int64_t)i * n + i] += d[j];
}

size_t node_partial_elems() { return (size_t)(2 * FGFRFT_SMS) * (kCbA + kNdPairs * 64) + kNdPairs * 64; }

cudaError_t launch_add_diag(double* w, int n, int64_t stride, const double* d, int r, cudaStream_t stream) {
    add_diag_kernel<<<dim3((unsigned)((n + 255) / 256), (unsigned)r), 256, 0, stream>>>(w, n, stride, d, r);
    return cudaGetLastError();
}

template <bool MSE, int T>
static cudaError_t node_combine_t(int ctas, size_t smem, cudaStream_t st, const double* zin, const double* xc,
                                  int64_t count, int r, int rp, const double* pc, int n_alpha, double* y, double* lp,
                                  double* gp) {
    static PerDeviceOnce attr;
    if (cudaError_t e = attr.run([] {
            return cudaFuncSetAttribute(node_combine_kernel<MSE, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)node_smem_bytes(8 * T - 1));
        }))
        return e;
    node_combine_kernel<MSE, T><<<ctas, 256, smem, st>>>(zin, xc, count, r, rp, pc, n_alpha, y, lp, gp);
    return cudaGetLastError();
}

template <bool MSE>
static cudaError_t node_combine_dispatch(int t8, int ctas, size_t smem, cudaStream_t st, const double* zin,
                                         const double* xc, int64_t count, int r, int rp, const double* pc,
                                         int n_alpha, double* y, double* lp, double* gp) {
    switch (t8) {
#define FGB_ND(T) \
    case T: return node_combine_t<MSE, T>(ctas, smem, st, zin, xc, count, r, rp, pc, n_alpha, y, lp, gp);
        FGB_ND(1) FGB_ND(2) FGB_ND(3) FGB_ND(4) FGB_ND(5) FGB_ND(6) FGB_ND(7)
#undef FGB_ND
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_node_combine(const double* zin, const double* xc, int64_t count, int r, int rp, const double* pc,
                                int n_alpha, double* y, double* partial, double norm, double* loss, double* dlda,
                                cudaStream_t stream) {
    if (n_alpha > kCbA || r > kNdMaxR || rp > kNdMaxR || rp % 4 || r > rp) return cudaErrorInvalidValue;
    const int64_t nch = (count + kNdP - 1) / kNdP;
    const int ctas = (int)(nch < 2 * FGFRFT_SMS ? nch : 2 * FGFRFT_SMS);
    const size_t smem = node_smem_bytes(r);
    const int t8 = node_rows8(r) / 8;
    cudaError_t e = cudaSuccess;
    if (!xc) {
        e = node_combine_dispatch<false>(t8, ctas, smem, stream, zin, nullptr, count, r, rp, pc, n_alpha, y, nullptr,
                                         nullptr);
        return e;
    }
    double* lp = partial;
    double* gp = partial + (size_t)ctas * kCbA;
    double* gs = gp + (size_t)ctas * kNdPairs * 64;
    e = node_combine_dispatch<true>(t8, ctas, smem, stream, zin, xc, count, r, rp, pc, n_alpha, y, lp, gp);
    if (e != cudaSuccess) return e;
    const int elems = t8 * (t8 + 1) / 2 * 64;
    node_gram_reduce_kernel<<<(elems + 31) / 32, 512, 0, stream>>>(gp, ctas, elems, gs);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    node_reduce_kernel<<<n_alpha, 128, 0, stream>>>(lp, gs, ctas, r, rp, pc, n_alpha, norm, loss, dlda);
    return cudaGetLastError();
}

}  // namespace fgb
