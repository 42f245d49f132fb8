// layout.cu -- conversion between the API's column-major matrices and the tiled, swizzled
// device layout of the power cache (see common.cuh), with optional complex64 demotion.
#include "common.cuh"

namespace fgb {

// dst tiled (padded with zeros) <- src column-major n x n (ld = n).
template <typename S, typename D>
__global__ void __launch_bounds__(256) to_tiled_kernel(const S* __restrict__ src, D* __restrict__ dst, int n, int nt) {
    const int I = blockIdx.x % nt, J = blockIdx.x / nt;
    const int r = threadIdx.x & 31, w = threadIdx.x >> 5;
    D* t = dst + tile_base(I, J, nt);
    const int row = I * kTile + r;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int c = w + 8 * i, col = J * kTile + c;
        D v;
        if (row < n && col < n) {
            const S x = src[(int64_t)col * n + row];
            v.x = x.x;
            v.y = x.y;
        } else {
            v.x = 0;
            v.y = 0;
        }
        t[swz(r, c)] = v;
    }
}

template <typename S>
__global__ void __launch_bounds__(256) from_tiled_kernel(const S* __restrict__ src, double2* __restrict__ dst, int n, int nt) {
    const int I = blockIdx.x % nt, J = blockIdx.x / nt;
    const int r = threadIdx.x & 31, w = threadIdx.x >> 5;
    const S* t = src + tile_base(I, J, nt);
    const int row = I * kTile + r;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int c = w + 8 * i, col = J * kTile + c;
        if (row < n && col < n) {
            const S v = t[swz(r, c)];
            dst[(int64_t)col * n + row] = make_double2((double)v.x, (double)v.y);
        }
    }
}

// elem_bytes_dst: 16 (complex128 tiles) or 8 (complex64 tiles); src is always complex128.
cudaError_t launch_to_tiled(const void* src, void* dst, int n, int elem_bytes_dst, cudaStream_t stream) {
    const int nt = (int)ceil_div(n, kTile);
    if (elem_bytes_dst == 16)
        to_tiled_kernel<double2, double2><<<nt * nt, 256, 0, stream>>>((const double2*)src, (double2*)dst, n, nt);
    else
        to_tiled_kernel<double2, float2><<<nt * nt, 256, 0, stream>>>((const double2*)src, (float2*)dst, n, nt);
    return cudaGetLastError();
}

cudaError_t launch_from_tiled(const void* src, void* dst, int n, int elem_bytes_src, cudaStream_t stream) {
    const int nt = (int)ceil_div(n, kTile);
    if (elem_bytes_src == 16)
        from_tiled_kernel<double2><<<nt * nt, 256, 0, stream>>>((const double2*)src, (double2*)dst, n, nt);
    else
        from_tiled_kernel<float2><<<nt * nt, 256, 0, stream>>>((const float2*)src, (double2*)dst, n, nt);
    return cudaGetLastError();
}

}  // namespace fgb
