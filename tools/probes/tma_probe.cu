// Per-SM streaming bandwidth probe (B200): how many bytes/s can g SMs pull from HBM with
// (a) a TMA bulk-copy ring (one producer lane, chunk bytes, S stages; consumer just releases), or
// (b) plain 128-bit loads by all warps (unrolled). Used to size the synthesis / GEMM SM split.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu && ./tma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, int c) { asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mexpect(uint64_t* b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void marrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}

__global__ void tma_kernel(const unsigned char* src, int64_t chunks, int chunk, int stages, int nprod) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * chunk);
    uint64_t* empty = full + stages;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // nprod independent rings (one per producer warp), stages split between them
    const int sp = stages / nprod;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { minit(full + s, 1); minit(empty + s, 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int ring = w >> 1;  // warps 2r (producer), 2r + 1 (consumer)
    if (ring >= nprod || lane) return;
    const int64_t per = (chunks + (int64_t)gridDim.x * nprod - 1) / ((int64_t)gridDim.x * nprod);
    const int64_t c0 = ((int64_t)blockIdx.x * nprod + ring) * per;
    const int64_t c1 = c0 + per < chunks ? c0 + per : chunks;
    uint64_t* f = full + ring * sp;
    uint64_t* e = empty + ring * sp;
    unsigned char* buf = sm + (size_t)ring * sp * chunk;
    if ((w & 1) == 0) {
        int it = 0;
        for (int64_t c = c0; c < c1; ++c, ++it) {
            const int s = it % sp;
            if (it >= sp) mwait(e + s, ((it / sp) - 1) & 1);
            mexpect(f + s, chunk);
            bulk(buf + (size_t)s * chunk, src + c * chunk, chunk, f + s);
        }
    } else {
        int it = 0;
        for (int64_t c = c0; c < c1; ++c, ++it) {
            const int s = it % sp;
            mwait(f + s, (it / sp) & 1);
            marrive(e + s);
        }
    }
}

__global__ void ldg_kernel(const uint4* src, int64_t n16, unsigned long long* sink) {
    uint32_t acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n16; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
    const size_t bytes = (size_t)6 << 30;
    unsigned char* src;
    unsigned long long* sink;
    cudaMalloc(&src, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(src, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    const int grids[] = {8, 20, 40, 60, 80, 148};
    struct Cfg { int chunk, stages, nprod; } cfgs[] = {
        {40960, 4, 1}, {40960, 5, 1}, {20480, 10, 1}, {10240, 16, 1}, {10240, 20, 2}, {10240, 20, 4}, {20480, 10, 2}, {4096, 48, 4}};
    for (const Cfg& c : cfgs) {
        const int smem = c.chunk * c.stages + 2 * c.stages * 8;
        for (int g : grids) {
            const int64_t chunks = bytes / c.chunk;
            tma_kernel<<<g, 64 * c.nprod, smem>>>(src, chunks, c.chunk, c.stages, c.nprod);
            cudaEventRecord(a);
            tma_kernel<<<g, 64 * c.nprod, smem>>>(src, chunks, c.chunk, c.stages, c.nprod);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double gbs = chunks * (double)c.chunk / (ms * 1e-3) / 1e9;
            printf("tma chunk %6d stages %2d prod %d grid %3d: %8.1f GB/s  (%6.1f GB/s per SM)  err %s\n", c.chunk,
                   c.stages, c.nprod, g, gbs, gbs / g, cudaGetErrorString(cudaGetLastError()));
        }
    }
    for (int th : {256, 512, 1024})
        for (int g : grids) {
            const int64_t n16 = bytes / 16;
            ldg_kernel<<<g, th>>>((const uint4*)src, n16, sink);
            cudaEventRecord(a);
            ldg_kernel<<<g, th>>>((const uint4*)src, n16, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double gbs = bytes / (ms * 1e-3) / 1e9;
            printf("ldg threads %4d grid %3d: %8.1f GB/s  (%6.1f GB/s per SM)\n", th, g, gbs, gbs / g);
        }
    return 0;
}
