// store.cu -- device side of the on-disk power cache: an order-independent
// 64-bit checksum of the resident slabs, written at save and re-checked after a load.
#include "common.cuh"

namespace fgb {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// out += sum_p mix64(w[p] + p * golden) (wrapping): position-dependent, summation order free,
// so the value does not depend on the grid.
__global__ void __launch_bounds__(256) checksum_kernel(const uint64_t* __restrict__ w, int64_t count,
                                                       unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < count; p += (int64_t)gridDim.x * blockDim.x)
        acc += mix64(w[p] + (uint64_t)p * 0x9E3779B97F4A7C15ull);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

cudaError_t launch_checksum(const void* data, size_t bytes, unsigned long long* out, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    checksum_kernel<<<4 * FGFRFT_SMS, 256, 0, st>>>(static_cast<const uint64_t*>(data), (int64_t)(bytes / 8), out);
    return cudaGetLastError();
}

}  // namespace fgb
