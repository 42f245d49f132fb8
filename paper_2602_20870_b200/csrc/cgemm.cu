// cgemm.cu -- complex64 GEMM for the complex64 cache path (BASELINE config 3 c64):
//
//   C[b] (M x N) = op(A[b]) * op(B[b]) (+ C[b]), column-major complex64, op in {X, X^H}.
//
// FP32 FFMA on the CUDA cores: complex64 results must come within 1e-4 of the fp64 oracle
// (north star), which single-pass TF32 cannot guarantee at K = 4096 (SURVEY 7 "hard parts"),
// and tcgen05 has no fp32-input kind. CTA tile 128 x 64 complex, BK = 16, 256 threads with
// 8 x 4 complex accumulators each (rows tm*4+{0..3} and 64+tm*4+{0..3}, cols tn*2+{0,1} and
// 32+tn*2+{0,1}); operands are staged global -> registers -> shared with the conjugation folded
// into the stored values, double-buffered.
#include "common.cuh"

namespace fgb {

constexpr int kCgBM = 128, kCgBN = 64, kCgBK = 16;

template <bool CA, bool CB>
__global__ void __launch_bounds__(256, 2)
cgemm_kernel(int M, int N, int K, const float2* __restrict__ A, int64_t lda, int64_t sA, const float2* __restrict__ B,
             int64_t ldb, int64_t sB, float2* __restrict__ Cm, int64_t ldc, int64_t sC, int accumulate) {
    __shared__ __align__(16) float2 As[2][kCgBK][kCgBM];
    __shared__ __align__(16) float2 Bs[2][kCgBK][kCgBN];
    const int bz = blockIdx.z;
    A += bz * sA;
    B += bz * sB;
    Cm += bz * sC;
    const int m0 = blockIdx.x * kCgBM, n0 = blockIdx.y * kCgBN;
    const int tid = threadIdx.x, tm = tid & 15, tn = tid >> 4;

    // Each thread stages 8 elements of A and 4 of B per K tile.
    float2 ra[8], rb[4];
    auto gload = [&](int k0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int idx = tid + 256 * j;  // 0..2047 over the 16 x 128 A tile
            int k, m;
            if (!CA) { k = idx / kCgBM; m = idx % kCgBM; }   // A(m, k) at m + k*lda: m fastest
            else { m = idx / kCgBK; k = idx % kCgBK; }       // A^H: stored A_st(k, m) at k + m*lda
            const bool v = (m0 + m < M) && (k0 + k < K);
            float2 x = make_float2(0.f, 0.f);
            if (v) x = CA ? A[(int64_t)(m0 + m) * lda + k0 + k] : A[(int64_t)(k0 + k) * lda + m0 + m];
            if (CA) x.y = -x.y;
            ra[j] = x;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int idx = tid + 256 * j;  // 0..1023 over the 16 x 64 B tile
            int k, n;
            if (!CB) { n = idx / kCgBK; k = idx % kCgBK; }   // B(k, n) at k + n*ldb: k fastest
            else { k = idx / kCgBN; n = idx % kCgBN; }       // B^H: stored B_st(n, k) at n + k*ldb
            const bool v = (n0 + n < N) && (k0 + k < K);
            float2 x = make_float2(0.f, 0.f);
            if (v) x = CB ? B[(int64_t)(k0 + k) * ldb + n0 + n] : B[(int64_t)(n0 + n) * ldb + k0 + k];
            if (CB) x.y = -x.y;
            rb[j] = x;
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int idx = tid + 256 * j;
            int k, m;
            if (!CA) { k = idx / kCgBM; m = idx % kCgBM; }
            else { m = idx / kCgBK; k = idx % kCgBK; }
            As[buf][k][m] = ra[j];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int idx = tid + 256 * j;
            int k, n;
            if (!CB) { n = idx / kCgBK; k = idx % kCgBK; }
            else { k = idx / kCgBN; n = idx % kCgBN; }
            Bs[buf][k][n] = rb[j];
        }
    };

    float acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.f;

    const int nk = (K + kCgBK - 1) / kCgBK;
    gload(0);
    sstore(0);
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) gload((kt + 1) * kCgBK);
#pragma unroll
        for (int kk = 0; kk < kCgBK; ++kk) {
            float2 a[8], b[4];
            const float4* pa0 = reinterpret_cast<const float4*>(&As[buf][kk][tm * 4]);
            const float4* pa1 = reinterpret_cast<const float4*>(&As[buf][kk][64 + tm * 4]);
            float4 v;
            v = pa0[0]; a[0] = make_float2(v.x, v.y); a[1] = make_float2(v.z, v.w);
            v = pa0[1]; a[2] = make_float2(v.x, v.y); a[3] = make_float2(v.z, v.w);
            v = pa1[0]; a[4] = make_float2(v.x, v.y); a[5] = make_float2(v.z, v.w);
            v = pa1[1]; a[6] = make_float2(v.x, v.y); a[7] = make_float2(v.z, v.w);
            v = *reinterpret_cast<const float4*>(&Bs[buf][kk][tn * 2]);
            b[0] = make_float2(v.x, v.y); b[1] = make_float2(v.z, v.w);
            v = *reinterpret_cast<const float4*>(&Bs[buf][kk][32 + tn * 2]);
            b[2] = make_float2(v.x, v.y); b[3] = make_float2(v.z, v.w);
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    acc[i][j][0] = fmaf(a[i].x, b[j].x, acc[i][j][0]);
                    acc[i][j][0] = fmaf(-a[i].y, b[j].y, acc[i][j][0]);
                    acc[i][j][1] = fmaf(a[i].x, b[j].y, acc[i][j][1]);
                    acc[i][j][1] = fmaf(a[i].y, b[j].x, acc[i][j][1]);
                }
        }
        if (kt + 1 < nk) {
            sstore(buf ^ 1);
            __syncthreads();
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int row = m0 + (i < 4 ? tm * 4 + i : 64 + tm * 4 + (i - 4));
        if (row >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int col = n0 + (j < 2 ? tn * 2 + j : 32 + tn * 2 + (j - 2));
            if (col >= N) continue;
            float2* dst = Cm + (int64_t)col * ldc + row;
            float2 r = make_float2(acc[i][j][0], acc[i][j][1]);
            if (accumulate) {
                const float2 o = *dst;
                r.x += o.x;
                r.y += o.y;
            }
            *dst = r;
        }
    }
}

cudaError_t launch_cgemm(int M, int N, int K, const void* A, int64_t lda, int64_t sA, bool conj_a, const void* B,
                         int64_t ldb, int64_t sB, bool conj_b, void* C, int64_t ldc, int64_t sC, int batch,
                         bool accumulate, cudaStream_t stream) {
    if (M <= 0 || N <= 0 || batch <= 0) return cudaSuccess;
    const dim3 grid((unsigned)ceil_div(M, kCgBM), (unsigned)ceil_div(N, kCgBN), (unsigned)batch);
#define FGB_CG_CASE(CA, CB)                                                                                 \
    cgemm_kernel<CA, CB><<<grid, 256, 0, stream>>>(M, N, K, (const float2*)A, lda, sA, (const float2*)B, ldb, \
                                                   sB, (float2*)C, ldc, sC, accumulate ? 1 : 0)
    if (!conj_a && !conj_b) FGB_CG_CASE(false, false);
    else if (conj_a && !conj_b) FGB_CG_CASE(true, false);
    else if (!conj_a && conj_b) FGB_CG_CASE(false, true);
    else FGB_CG_CASE(true, true);
#undef FGB_CG_CASE
    return cudaGetLastError();
}

__global__ void promote_kernel(const float2* __restrict__ src, double2* __restrict__ dst, int64_t count) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 v = src[i];
        dst[i] = make_double2((double)v.x, (double)v.y);
    }
}

cudaError_t launch_promote(const void* src, void* dst, int64_t count, cudaStream_t stream) {
    promote_kernel<<<8 * FGFRFT_SMS, 256, 0, stream>>>((const float2*)src, (double2*)dst, count);
    return cudaGetLastError();
}

}  // namespace fgb
