// zgemm.cu -- complex128 GEMM on the FP64 tensor cores (DMMA.8x8x4) for sm_100a.
//
//   C[b] (M x N) = op(A[b]) * op(B[b])   (+ C[b] if accumulate), column-major complex128,
//   op(A) = A or A^H, op(B) = B or B^H.
//
// tcgen05 has no f64 kind, so on B200 the FP64 tensor path is the warp-level mma.sync DMMA
// (measured 37.1 TFLOP/s, profiles/r01_fp64_peaks.json). Used by:
//   K1 power-cache builder   P_k = F P_{k-1}          (transform.hpp:58)
//   K3 apply                 Y = Q X, Q^H X           (transform.hpp:140, 147)
//   K4 dL/dalpha             M = G X^H                (learn.hpp:88-92 restated as Re<M, F^k>)
//
// CTA tile 128 x 64 complex, BK = 16, 8 warps as 4 (m) x 2 (n), warp tile 32 x 32 complex =
// 4 x 4 blocks of 8x8; a complex 8x8x4 step is four real DMMAs. 3-stage cp.async ring; shared
// layouts are padded so every fragment load (LDS.128) is bank-conflict free.
#include "common.cuh"

namespace fgb {

constexpr int kGemmBM = 128, kGemmBN = 64, kGemmBK = 16, kGemmStages = 3, kGemmThreads = 256;
constexpr int kLdMK = kGemmBM + 2;  // A tile stored [k][m]  (A not conjugated)
constexpr int kLdKM = kGemmBK + 4;  // A tile stored [m][k]  (A^H) and B tile [n][k] (B)
constexpr int kLdNK = kGemmBN + 2;  // B tile stored [k][n]  (B^H)

template <bool CA>
constexpr int a_stage_elems() { return CA ? kGemmBM * kLdKM : kGemmBK * kLdMK; }
template <bool CB>
constexpr int b_stage_elems() { return CB ? kGemmBK * kLdNK : kGemmBN * kLdKM; }

template <bool CA, bool CB>
constexpr size_t gemm_smem_bytes() {
    return (size_t)kGemmStages * (a_stage_elems<CA>() + b_stage_elems<CB>()) * sizeof(double2);
}

template <bool CA, bool CB>
__global__ void __launch_bounds__(kGemmThreads, 1)
zgemm_dmma_kernel(int M, int N, int K, const double2* __restrict__ A, int64_t lda, int64_t sA,
                  const double2* __restrict__ B, int64_t ldb, int64_t sB, double2* __restrict__ Cm,
                  int64_t ldc, int64_t sC, int accumulate) {
    extern __shared__ __align__(128) unsigned char smem[];
    double2* As = reinterpret_cast<double2*>(smem);
    double2* Bs = As + kGemmStages * a_stage_elems<CA>();

    const int bz = blockIdx.z;
    A += bz * sA;
    B += bz * sB;
    Cm += bz * sC;
    const int m0 = blockIdx.x * kGemmBM, n0 = blockIdx.y * kGemmBN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 3, wn = warp >> 2;
    const int g = lane >> 2, t = lane & 3;
    const int nk = (K + kGemmBK - 1) / kGemmBK;

    auto load_stage = [&](int kt, int s) {
        const int k0 = kt * kGemmBK;
        double2* as = As + s * a_stage_elems<CA>();
        double2* bs = Bs + s * b_stage_elems<CB>();
        if (!CA) {  // A stored M x K: tile columns k, m contiguous -> smem [k][m]
#pragma unroll
            for (int j = 0; j < (kGemmBM * kGemmBK) / kGemmThreads; ++j) {
                const int idx = tid + j * kGemmThreads;
                const int k = idx / kGemmBM, m = idx % kGemmBM;
                const bool v = (m0 + m < M) && (k0 + k < K);
                const double2* src = v ? A + (int64_t)(k0 + k) * lda + (m0 + m) : A;
                cp_async16(as + k * kLdMK + m, src, v);
            }
        } else {    // A stored K x M: tile columns m, k contiguous -> smem [m][k]
#pragma unroll
            for (int j = 0; j < (kGemmBM * kGemmBK) / kGemmThreads; ++j) {
                const int idx = tid + j * kGemmThreads;
                const int m = idx / kGemmBK, k = idx % kGemmBK;
                const bool v = (m0 + m < M) && (k0 + k < K);
                const double2* src = v ? A + (int64_t)(m0 + m) * lda + (k0 + k) : A;
                cp_async16(as + m * kLdKM + k, src, v);
            }
        }
        if (!CB) {  // B stored K x N: columns n, k contiguous -> smem [n][k]
#pragma unroll
            for (int j = 0; j < (kGemmBN * kGemmBK) / kGemmThreads; ++j) {
                const int idx = tid + j * kGemmThreads;
                const int n = idx / kGemmBK, k = idx % kGemmBK;
                const bool v = (n0 + n < N) && (k0 + k < K);
                const double2* src = v ? B + (int64_t)(n0 + n) * ldb + (k0 + k) : B;
                cp_async16(bs + n * kLdKM + k, src, v);
            }
        } else {    // B stored N x K: columns k, n contiguous -> smem [k][n]
#pragma unroll
            for (int j = 0; j < (kGemmBN * kGemmBK) / kGemmThreads; ++j) {
                const int idx = tid + j * kGemmThreads;
                const int k = idx / kGemmBN, n = idx % kGemmBN;
                const bool v = (n0 + n < N) && (k0 + k < K);
                const double2* src = v ? B + (int64_t)(k0 + k) * ldb + (n0 + n) : B;
                cp_async16(bs + k * kLdNK + n, src, v);
            }
        }
    };

    double acc[4][4][4];  // [mb][nb][re0, re1, im0, im1]
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.0;

#pragma unroll
    for (int s = 0; s < kGemmStages - 1; ++s) {
        if (s < nk) load_stage(s, s);
        cp_async_commit();
    }

    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<kGemmStages - 2>();
        __syncthreads();
        {
            const int nxt = kt + kGemmStages - 1;
            if (nxt < nk) load_stage(nxt, nxt % kGemmStages);
            cp_async_commit();
        }
        const int s = kt % kGemmStages;
        const double2* as = As + s * a_stage_elems<CA>();
        const double2* bs = Bs + s * b_stage_elems<CB>();
#pragma unroll
        for (int kk = 0; kk < kGemmBK; kk += 4) {
            double ar[4], ai[4], nai[4], br[4], bi[4];
#pragma unroll
            for (int mb = 0; mb < 4; ++mb) {
                const int m = wm * 32 + mb * 8 + g;
                const double2 v = CA ? as[m * kLdKM + kk + t] : as[(kk + t) * kLdMK + m];
                ar[mb] = v.x;
                ai[mb] = CA ? -v.y : v.y;
                nai[mb] = -ai[mb];
            }
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) {
                const int n = wn * 32 + nb * 8 + g;
                const double2 v = CB ? bs[(kk + t) * kLdNK + n] : bs[n * kLdKM + kk + t];
                br[nb] = v.x;
                bi[nb] = CB ? -v.y : v.y;
            }
#pragma unroll
            for (int mb = 0; mb < 4; ++mb)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) {
                    double* c = acc[mb][nb];
                    dmma884(c[0], c[1], ar[mb], br[nb]);
                    dmma884(c[0], c[1], nai[mb], bi[nb]);
                    dmma884(c[2], c[3], ar[mb], bi[nb]);
                    dmma884(c[2], c[3], ai[mb], br[nb]);
                }
        }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int mb = 0; mb < 4; ++mb) {
        const int row = m0 + wm * 32 + mb * 8 + g;
        if (row >= M) continue;
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int col = n0 + wn * 32 + nb * 8 + 2 * t + j;
                if (col >= N) continue;
                double2* dst = Cm + (int64_t)col * ldc + row;
                double2 v = make_double2(acc[mb][nb][j], acc[mb][nb][2 + j]);
                if (accumulate) {
                    const double2 o = *dst;
                    v.x += o.x;
                    v.y += o.y;
                }
                *dst = v;
            }
        }
    }
}

// C = op(A) op(B) (+C). conj_a: A stored K x M and op(A) = A^H; conj_b: B stored N x K.
cudaError_t launch_zgemm(int M, int N, int K, const void* A, int64_t lda, int64_t sA, bool conj_a,
                         const void* B, int64_t ldb, int64_t sB, bool conj_b, void* C, int64_t ldc,
                         int64_t sC, int batch, bool accumulate, cudaStream_t stream) {
    if (M <= 0 || N <= 0 || batch <= 0) return cudaSuccess;
    const dim3 grid((unsigned)ceil_div(M, kGemmBM), (unsigned)ceil_div(N, kGemmBN), (unsigned)batch);
#define FGB_GEMM_CASE(CA, CB)                                                                                \
    {                                                                                                        \
        auto kern = zgemm_dmma_kernel<CA, CB>;                                                               \
        const size_t smem = gemm_smem_bytes<CA, CB>();                                                       \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e != cudaSuccess) return e;                                                                      \
        kern<<<grid, kGemmThreads, smem, stream>>>(M, N, K, (const double2*)A, lda, sA, (const double2*)B,   \
                                                   ldb, sB, (double2*)C, ldc, sC, accumulate ? 1 : 0);       \
    }
    if (!conj_a && !conj_b) FGB_GEMM_CASE(false, false)
    else if (conj_a && !conj_b) FGB_GEMM_CASE(true, false)
    else if (!conj_a && conj_b) FGB_GEMM_CASE(false, true)
    else FGB_GEMM_CASE(true, true)
#undef FGB_GEMM_CASE
    return cudaGetLastError();
}

}  // namespace fgb
