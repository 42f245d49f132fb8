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
    return ((size_t)kCbA * cb_ldc(tp) + (size_t)tp * kCbLdP + (size_t)kCbA * kCbLdP + kCbP) * sizeof(double);
}

int combine_max_terms() { return kCbMaxT; }

// z: 2L blocks of `count` doubles: block j < L holds F^(j+1) X, block L + j holds F^-(j+1) X.
template <bool STORE_Y>
__global__ void __launch_bounds__(256, 1)
combine_kernel(const double* __restrict__ z, const double* __restrict__ x, const double* __restrict__ xc,
               int64_t count, int l, int tp, const double* __restrict__ coef, int n_alpha, double g_scale,
               double* __restrict__ y, double* __restrict__ spart, double* __restrict__ lpart) {
    extern __shared__ __align__(16) double sm[];
    const int ldc = cb_ldc(tp);
    double* cf = sm;                       // [64][ldc]   coefficients c_aq (zero padded)
    double* zc = cf + kCbA * ldc;          // [tp][68]    chunk of every term
    double* gs = zc + tp * kCbLdP;         // [64][68]    G chunk
    double* xs = gs + kCbA * kCbLdP;       // [64]        Xc chunk
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    const int T = 2 * l + 1;

    for (int idx = tid; idx < kCbA * ldc; idx += 256) {
        const int a = idx / ldc, q = idx - a * ldc;
        cf[idx] = (a < n_alpha && q < T) ? coef[(int64_t)a * T + q] : 0.0;
    }
    for (int idx = tid; idx < (tp - T) * kCbLdP; idx += 256) zc[T * kCbLdP + idx] = 0.0;

    double sacc[kCbMaxT / 8][2];
    const int nqb = tp / 8;
#pragma unroll
    for (int qb = 0; qb < kCbMaxT / 8; ++qb) sacc[qb][0] = sacc[qb][1] = 0.0;
    double lacc = 0.0;  // sum of R^2 over this thread's (order g of warp, positions)

    const int64_t nchunks = (count + kCbP - 1) / kCbP;
    for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const int64_t p0 = ch * kCbP;
        const int pv = (int)((count - p0) < kCbP ? (count - p0) : kCbP);
        __syncthreads();  // previous chunk's readers are done
        // stage the chunk of every term (16-byte cp.async; count is a multiple of 2)
        for (int idx = tid; idx < T * (kCbP / 2); idx += 256) {
            const int q = idx / (kCbP / 2), c2 = idx - q * (kCbP / 2);
            const double* src;
            if (q == l) src = x;
            else if (q > l) src = z + (int64_t)(q - l - 1) * count;
            else src = z + (int64_t)(l + (l - q) - 1) * count;
            const bool v = 2 * c2 < pv;
            cp_async16(zc + q * kCbLdP + 2 * c2, src + p0 + (v ? 2 * c2 : 0), v);
        }
        if (tid < kCbP / 2) cp_async16(xs + 2 * tid, xc + p0 + (2 * tid < pv ? 2 * tid : 0), 2 * tid < pv);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();

        // Y (orders 8w..8w+7) x (64 positions) = C Z_chunk
        double yacc[8][2];
#pragma unroll
        for (int pb = 0; pb < 8; ++pb) yacc[pb][0] = yacc[pb][1] = 0.0;
        const double* crow = cf + (8 * warp + g) * ldc;
        for (int q0 = 0; q0 < tp; q0 += 4) {
            const double av = crow[q0 + t];
            const double* zrow = zc + (q0 + t) * kCbLdP + g;
#pragma unroll
            for (int pb = 0; pb < 8; ++pb) dmma884(yacc[pb][0], yacc[pb][1], av, zrow[8 * pb]);
        }
        // residual, loss, G; optional Y store
        const int a = 8 * warp + g;
#pragma unroll
        for (int pb = 0; pb < 8; ++pb) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int p = 8 * pb + 2 * t + e;
                const bool ok = p < pv && a < n_alpha;
                const double r = ok ? yacc[pb][e] - xs[p] : 0.0;
                lacc += r * r;
                gs[a * kCbLdP + p] = r * g_scale;
                if (STORE_Y && ok) y[(int64_t)a * count + p0 + p] = yacc[pb][e];
            }
        }
        __syncthreads();
        // S (orders 8w..8w+7) x (terms) += G_chunk Z_chunk^T
        const double* grow = gs + (8 * warp + g) * kCbLdP;
        for (int p4 = 0; p4 < kCbP; p4 += 4) {
            const double av = grow[p4 + t];
            const double* zcol = zc + g * kCbLdP + p4 + t;
#pragma unroll
            for (int qb = 0; qb < kCbMaxT / 8; ++qb)
                if (qb < nqb) dmma884(sacc[qb][0], sacc[qb][1], av, zcol[8 * qb * kCbLdP]);
        }
    }
    // partials: spart[cta][a][q] (q < tp), lpart[cta][a]
    double* sp = spart + (int64_t)blockIdx.x * kCbA * tp;
    const int a = 8 * warp + g;
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
    if (idx < n_alpha) {
        double acc = 0.0;
        for (int c = 0; c < ctas; ++c) acc += lpart[(int64_t)c * kCbA + idx];
        loss[idx] = acc * norm;
    }
}

int combine_ctas() { return FGFRFT_SMS; }

size_t combine_partial_elems(int tp) { return (size_t)FGFRFT_SMS * kCbA * (tp + 1); }

// n_alpha <= 64, 2l + 1 <= 136; count = 2 N B (even). spart >= combine_partial_elems doubles.
cudaError_t launch_combine(const double* z, const double* x, const double* xc, int64_t count, int l,
                           const double* coef, int n_alpha, double norm, double* y, double* partial, double* s,
                           double* loss, cudaStream_t stream) {
    const int T = 2 * l + 1, tp = (T + 7) / 8 * 8;
    if (n_alpha < 1 || n_alpha > kCbA || tp > kCbMaxT || count % 2) return cudaErrorInvalidValue;
    const size_t smem = combine_smem_bytes(tp);
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(combine_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)combine_smem_bytes(kCbMaxT));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(combine_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)combine_smem_bytes(kCbMaxT));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int64_t nchunks = (count + kCbP - 1) / kCbP;
    const int ctas = (int)(nchunks < FGFRFT_SMS ? nchunks : FGFRFT_SMS);
    double* spart = partial;
    double* lpart = partial + (size_t)ctas * kCbA * tp;
    if (y)
        combine_kernel<true><<<ctas, 256, smem, stream>>>(z, x, xc, count, l, tp, coef, n_alpha, 2.0 * norm, y, spart,
                                                          lpart);
    else
        combine_kernel<false><<<ctas, 256, smem, stream>>>(z, x, xc, count, l, tp, coef, n_alpha, 2.0 * norm, y,
                                                           spart, lpart);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int threads = 256, blocks = (n_alpha * T + threads - 1) / threads;
    combine_reduce_kernel<<<blocks, threads, 0, stream>>>(spart, lpart, ctas, tp, T, n_alpha, norm, s, loss);
    return cudaGetLastError();
}

}  // namespace fgb
