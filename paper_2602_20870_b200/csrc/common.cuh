// common.cuh -- sm_100a device helpers shared by the FGFRFT kernels.
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>

#ifndef FGFRFT_SMS
#define FGFRFT_SMS 148
#endif

namespace fgb {

// Complex element types: (re, im) interleaved, 16 B (c128) or 8 B (c64).
template <typename R> struct cplx;
template <> struct cplx<double> { using type = double2; };
template <> struct cplx<float> { using type = float2; };
template <typename R> using cplx_t = typename cplx<R>::type;

// ---------------------------------------------------------------- mbarrier / bulk copy (TMA)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// 1-D bulk async copy global -> shared (UBLKCP), completion counted on `bar` in bytes.
// dst, src 16-B aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Same with an L2 eviction-priority hint (evict_first for streamed cache slabs).
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// ---------------------------------------------------------------- cp.async (LDGSTS), 16 B

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    const int sz = valid ? 16 : 0;  // src-size 0 => zero fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
    const int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---------------------------------------------------------------- DMMA (FP64 tensor core)

// D(8x8) += A(8x4, row) * B(4x8, col). Lane (g = lane>>2, t = lane&3) holds
// a = A[g][t], b = B[t][g], d = {D[g][2t], D[g][2t+1]}.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- tiled cache layout
//
// Device slabs of the power cache are stored TILED: the n x n matrix is padded to
// npad = 32 * nt (zeros) and cut into 32x32 tiles; tile (I, J) occupies 1024 consecutive
// elements at ((J * nt + I) * 1024), and tile element (i, j) sits at j * 32 + (i ^ j).
// One tile = one contiguous TMA bulk copy (16 KB complex128), and the XOR swizzle makes both
// the direct read (lanes along i) and the transposed read (lanes along j) of a staged tile
// bank-conflict free without padding shared memory.
constexpr int kTile = 32;
constexpr int kTileElems = kTile * kTile;

__host__ __device__ __forceinline__ int64_t tile_base(int I, int J, int nt) {
    return ((int64_t)J * nt + I) * kTileElems;
}
__host__ __device__ __forceinline__ int swz(int i, int j) { return j * kTile + (i ^ j); }

// ---------------------------------------------------------------- device sinc (sinc.hpp:15-36)
// (device libm: within ~1 ulp of the host coefficients; used where orders live on the device)
__device__ __forceinline__ double dsinc(double x) {
    if (x == nearbyint(x)) return x == 0.0 ? 1.0 : 0.0;
    if (fabs(x) < 1e-6) {
        const double px = CUDART_PI * x;
        return 1.0 - px * px / 6.0;
    }
    return sin(CUDART_PI * x) / (CUDART_PI * x);
}
__device__ __forceinline__ double dsinc_deriv(double x) {
    if (x == nearbyint(x)) {
        if (x == 0.0) return 0.0;
        const long long k = (long long)x;
        return (k % 2 == 0 ? 1.0 : -1.0) / x;
    }
    if (fabs(x) < 1e-6) {
        const double pi2 = CUDART_PI * CUDART_PI;
        return -pi2 * x / 3.0 + pi2 * pi2 * x * x * x / 30.0;
    }
    const double px = CUDART_PI * x;
    return cos(px) / x - sin(px) / (CUDART_PI * x * x);
}

// ---------------------------------------------------------------- misc

// One-time per-DEVICE setup (cudaFuncSetAttribute opt-ins are per device): a bit per device,
// set with an atomic OR after the first success. Concurrent first calls may both run f (the
// attribute calls are idempotent); no unsynchronised static flag.
struct PerDeviceOnce {
    std::atomic<uint64_t> mask{0};
    template <class F>
    cudaError_t run(F&& f) {
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t bit = 1ull << (dev & 63);
        if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
        const cudaError_t e = f();
        if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_acq_rel);
        return e;
    }
};

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Pair index p -> (I, J) with I <= J, p = J(J+1)/2 + I.
__device__ __forceinline__ void pair_of(int p, int& I, int& J) {
    int j = static_cast<int>((sqrt(8.0 * p + 1.0) - 1.0) * 0.5);
    while (j * (j + 1) / 2 > p) --j;
    while ((j + 1) * (j + 2) / 2 <= p) ++j;
    J = j;
    I = p - j * (j + 1) / 2;
}

// I-major enumeration of the tile pairs (I <= J): row I's pairs are contiguous, so the pairs
// whose smaller tile index lies in [I0, I1) -- everything that completes rows [32 I0, 32 I1) of
// a synthesised operator -- are one index range [pairs_before(I0), pairs_before(I1)).
__host__ __device__ __forceinline__ int64_t pairs_before(int64_t I, int64_t nt) { return I * nt - I * (I - 1) / 2; }
__device__ __forceinline__ void pair_of_imajor(int p, int nt, int& I, int& J) {
    const double b = 2.0 * nt + 1.0;
    int i = (int)((b - sqrt(b * b - 8.0 * p)) * 0.5);
    i = max(0, min(i, nt - 1));
    while (i > 0 && pairs_before(i, nt) > p) --i;
    while (i + 1 < nt && pairs_before(i + 1, nt) <= p) ++i;
    I = i;
    J = i + (int)(p - pairs_before(i, nt));
}

// The order window's per-call interpolation weights (packed.cu window_synth_kernel, passed by value):
// rows [l_j(a) ..][l_j'(a) ..] over r <= kWindowMaxNodes node operators.
constexpr int kWindowMaxNodes = 48;
struct WindowWeights {
    double w[4][kWindowMaxNodes];
};

}  // namespace fgb
