// ops.cu -- small device kernels around the hot path: MSE residual / cotangent with a
// deterministic loss reduction, and complex128 -> complex64 demotion of cache slabs.
#include "common.cuh"

namespace fgb {

constexpr int kResBlocks = 4 * FGFRFT_SMS;  // per order, fixed -> deterministic partition

// For order a (blockIdx.y): R = Y_a - Xc, G_a = scale * R, loss partial per block = sum |R|^2
// (accumulated in double for both element types).
template <typename C>
__global__ void __launch_bounds__(256)
mse_residual_kernel(const C* __restrict__ y, const C* __restrict__ xc, int64_t count, double scale,
                    C* __restrict__ g, double* __restrict__ partial) {
    const int a = blockIdx.y;
    const C* ya = y + (int64_t)a * count;
    C* ga = g + (int64_t)a * count;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const C yv = ya[i], xv = xc[i];
        const double rx = (double)yv.x - (double)xv.x, ry = (double)yv.y - (double)xv.y;
        acc = fma(rx, rx, fma(ry, ry, acc));
        ga[i].x = scale * rx;
        ga[i].y = scale * ry;
    }
    __shared__ double wsum[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += wsum[w];
        partial[(int64_t)a * gridDim.x + blockIdx.x] = s;
    }
}

// out[a] = scale * sum_i partial[a][i]; fixed split over 128 threads + fixed tree (deterministic).
__global__ void __launch_bounds__(128) sum_rows_kernel(const double* __restrict__ partial, int cols, double scale,
                                                       double* __restrict__ out) {
    const double* row = partial + (int64_t)blockIdx.x * cols;
    double s = 0.0;
    for (int i = threadIdx.x; i < cols; i += 128) s += row[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ double ws[4];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = ((ws[0] + ws[1]) + (ws[2] + ws[3])) * scale;
}

size_t mse_partial_elems(int n_alpha) { return (size_t)n_alpha * kResBlocks; }

// loss_out[a] = ||Y_a - Xc||^2 * loss_scale ; g = g_scale (Y_a - Xc).
cudaError_t launch_mse_residual(const void* y, const void* xc, int64_t count, int n_alpha, double g_scale,
                                double loss_scale, void* g, double* partial, double* loss_out,
                                cudaStream_t stream, int elem_bytes) {
    if (elem_bytes == 16)
        mse_residual_kernel<double2><<<dim3(kResBlocks, n_alpha), 256, 0, stream>>>(
            (const double2*)y, (const double2*)xc, count, g_scale, (double2*)g, partial);
    else
        mse_residual_kernel<float2><<<dim3(kResBlocks, n_alpha), 256, 0, stream>>>(
            (const float2*)y, (const float2*)xc, count, g_scale, (float2*)g, partial);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    sum_rows_kernel<<<n_alpha, 128, 0, stream>>>(partial, kResBlocks, loss_scale, loss_out);
    return cudaGetLastError();
}

__global__ void demote_kernel(const double2* __restrict__ src, float2* __restrict__ dst, int64_t count) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const double2 v = src[i];
        dst[i] = make_float2((float)v.x, (float)v.y);
    }
}

cudaError_t launch_demote(const void* src, void* dst, int64_t count, cudaStream_t stream) {
    demote_kernel<<<8 * FGFRFT_SMS, 256, 0, stream>>>((const double2*)src, (float2*)dst, count);
    return cudaGetLastError();
}

// out[a] = sum_k dc[a][k] * s[a][k] in ascending k (dL/dalpha = sum_k c'_k s_k).
__global__ void coef_dot_kernel(const double* __restrict__ dc, const double* __restrict__ s, int n_alpha, int width,
                                double* __restrict__ out) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n_alpha) return;
    double acc = 0.0;
    for (int k = 0; k < width; ++k) acc += dc[(int64_t)a * width + k] * s[(int64_t)a * width + k];
    out[a] = acc;
}

cudaError_t launch_coef_dot(const double* dc, const double* s, int n_alpha, int width, double* out,
                            cudaStream_t stream) {
    coef_dot_kernel<<<(unsigned)ceil_div(n_alpha, 128), 128, 0, stream>>>(dc, s, n_alpha, width, out);
    return cudaGetLastError();
}

}  // namespace fgb
