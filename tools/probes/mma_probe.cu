// tcgen05.mma kind::i8 issue/throughput probe (B200): cycles per MMA for M in {64, 128}, N in
// {16 .. 256}, K = 32, operands in shared memory (content irrelevant), accumulate into TMEM.
// One CTA per SM, one thread issues R MMAs back to back, commit, wait; clock64 around.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu && ./mma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__global__ void probe(int m, int n, int reps, int issuers, long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar, bar2;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar2)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < issuers) {
        const int w = threadIdx.x >> 5;
        const uint32_t tm = tmem + (uint32_t)(w * 128);
        uint64_t* mybar = w == 0 ? &bar : &bar2;
        const uint32_t a0 = su32(sm), b0 = su32(sm + 65536);
        const uint32_t id = idesc(m, n);
        const long long t0 = clock64();
        for (int r = 0; r < reps / issuers; ++r) {
            const uint64_t ad = desc(a0 + (r & 7) * 4096, 128, 512), bd = desc(b0 + (r & 7) * 4096, 128, 512);
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tm), "l"(ad), "l"(bd), "r"(id), "r"(r));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(mybar)) : "memory");
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(mybar)) : "memory");
        const long long t1 = clock64();
        if (w == 0) out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
    const int reps = 4096;
    for (int iss : {1, 2})
    for (int m : {128})
        for (int n : {16, 64, 96, 128, 256}) {
            probe<<<148, 128, 140 * 1024>>>(m, n, reps, iss, d);
            probe<<<148, 128, 140 * 1024>>>(m, n, reps, iss, d);
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < 148; ++i) avg += h[i];
            avg /= 148;
            const double cyc = avg / reps;
            printf("issuers %d M %3d N %3d K 32: %7.1f clk per MMA  (%6.0f int8 MAC/clk/SM)  %s\n", iss, m, n, cyc, m * n * 32.0 / cyc,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
