// batch.cu -- K5: many small graphs at once (BASELINE config 5, the fractional-specformer shape:
// 4096 independent graphs, n <= 64, L = 16, H learnable orders per graph, C channels, complex64).
//
// One CTA per graph. Forward: the graph's L powers (tiled + swizzled, 32 KB each for n = 64)
// stream through a 4-stage TMA ring while 512 threads accumulate Q_h = c_0 I + sum_k a_hk P_k +
// b_hk P_k^H for all H heads in registers (each thread owns 8 elements x H heads; both P_ij and
// P_ji come from the same staged tile); Q_h then moves to shared memory and Y_h = Q_h X_g runs on
// the FP32 FFMA pipes from shared memory. Backward (dL/dalpha per graph and head): M_h = G_h X^H
// in registers (same element ownership), then one more pass over the powers forms
// s_hk = Re<M_h, P_k>, Re<M_h, P_k^H> with a transposing warp reduction, and
// dL/dalpha_h = sum_k c'_k s_hk. Coefficients for the 4096 x H orders are evaluated on the device
// (double precision, the sinc.hpp formulas; differences from glibc are ~1 ulp, far inside the
// complex64 tolerance), so a step has no host-side O(graphs x heads x L) work.
#include <math_constants.h>
#include <cstdlib>
#include <type_traits>

#include <cuda_bf16.h>

#include "common.cuh"
#include "tc.cuh"

namespace fgb {

constexpr int kBN = 64;          // padded graph size (2 x 2 tiles)
constexpr int kBTh = 512;        // threads per graph CTA
constexpr int kBStages = 4;      // power ring slots in region A for complex slabs (32 KB each)
constexpr int kBStagesR = 8;     // forward, real float slabs (16 KB each): the same 128 KB, twice the depth
constexpr int kBMaxHeads = 4;
constexpr int kBMaxCh = 64;
constexpr int kBSlab = 4 * kTileElems;  // elements per padded slab

// coef[o][2][2l+1] (c then dc) for every order o; heads > 0: also the FP32 copy the tcgen05 kernels
// stream, per graph [c_k | c_-k | c'_k | c'_-k][k = 0..l][4 heads] (one 16-byte load per power and
// table, heads padded to 4; tc_coef_stride floats), after the doubles.
__global__ void batch_coef_kernel(const double* __restrict__ alphas, int n_orders, int l, double* __restrict__ coef,
                                  float* __restrict__ coef_f, int heads, int fstride) {
    const int w = 2 * l + 1;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_orders * w) return;
    const int o = idx / w, t = idx % w;
    const double x = alphas[o] - (double)(t - l);
    const double c = dsinc(x), d = dsinc_deriv(x);
    coef[(size_t)o * 2 * w + t] = c;
    coef[(size_t)o * 2 * w + w + t] = d;
    if (coef_f) {
        float* f = coef_f + (size_t)(o / heads) * fstride + (o % heads);
        const int k = t - l, kk = k >= 0 ? k : -k, tb = k >= 0 ? 0 : 1, q = 4 * (l + 1);
        f[tb * q + 4 * kk] = (float)c;
        f[(2 + tb) * q + 4 * kk] = (float)d;
        if (k == 0) {
            f[q] = (float)c;
            f[3 * q] = (float)d;
        }
    }
}

// [G] column-major n x n complex128 (stride n*n) -> [G][slab k] tiled complex64 padded to 64
// (REAL: a real F's slabs as float, half the bytes and half the FMAs downstream).
template <bool REAL>
__global__ void __launch_bounds__(256) batch_to_tiled_kernel(const double2* __restrict__ src, int n, int l, int k,
                                                             void* __restrict__ dstv) {
    const int g = blockIdx.y, tile = blockIdx.x;  // tile = I + 2*J
    const int I = tile & 1, J = tile >> 1;
    const int r = threadIdx.x & 31, w = threadIdx.x >> 5;
    const double2* s = src + (int64_t)g * n * n;
    const int64_t off = ((int64_t)g * l + (k - 1)) * kBSlab + (int64_t)tile * kTileElems;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int c = w + 8 * i, row = I * 32 + r, col = J * 32 + c;
        double2 x = make_double2(0.0, 0.0);
        if (row < n && col < n) x = s[(int64_t)col * n + row];
        if (REAL)
            static_cast<float*>(dstv)[off + swz(r, c)] = (float)x.x;
        else
            static_cast<float2*>(dstv)[off + swz(r, c)] = make_float2((float)x.x, (float)x.y);
    }
}

// element (i, j) of a padded 64 x 64 tiled slab
__device__ __forceinline__ int bidx(int i, int j) { return ((j >> 5) * 2 + (i >> 5)) * kTileElems + swz(i & 31, j & 31); }

struct BatchSmem {
    // region A: TMA stages during the power passes, then Q_h / G_h; then X; then the mbarriers
    // and the per-power reduction table red[(l+1) x 16 warps x 8].
    static constexpr size_t kA = (size_t)kBStages * kBSlab * 8;          // 128 KB
    static constexpr size_t kX = (size_t)kBN * kBMaxCh * 8;              // 32 KB
    // + one more mbarrier (X / G bulk copy) before the table: forward keeps its coefficients there
    static size_t bytes(int l) { return kA + kX + (kBStagesR + 1) * 8 + (size_t)(l + 1) * 16 * 8 * 8 + 64; }
};

size_t batch_smem_bytes(int l) { return BatchSmem::bytes(l); }

// R: real slabs (a real F: Q real, half the bytes streamed and half the FMAs in both phases).
template <int H, bool R>
__global__ void __launch_bounds__(kBTh, 1)
batch_forward_kernel(const void* __restrict__ slabs, int n, int l, const double* __restrict__ coef,
                     const float2* __restrict__ x, int ch, float2* __restrict__ y) {
    using ST = typename std::conditional<R, float, float2>::type;  // slab / Q element
    extern __shared__ __align__(128) unsigned char smem[];
    ST* regA = reinterpret_cast<ST*>(smem);
    float2* xs = reinterpret_cast<float2*>(smem + BatchSmem::kA);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + BatchSmem::kA + BatchSmem::kX);
    constexpr int NS = R ? kBStagesR : kBStages;
    uint64_t* xbar = full + kBStagesR;
    const int g = blockIdx.x, tid = threadIdx.x;
    const int w = 2 * l + 1;
    float* cs = reinterpret_cast<float*>(xbar + 1);  // [h][w]: this graph's series coefficients
    const ST* gs = static_cast<const ST*>(slabs) + (int64_t)g * l * kBSlab;
    const uint32_t bytes = kBSlab * sizeof(ST);
    auto issue = [&](int k, int s) {
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(regA + (size_t)s * kBSlab, gs + (int64_t)(k - 1) * kBSlab, bytes, &full[s]);
    };
    // Full-size graphs (n = 64, 64 channels): X_g is one contiguous 32 KB block in the xs layout,
    // bulk-copied at kernel start; it is first needed by the Y phase, so the copy overlaps the
    // whole power pass instead of exposing a global-load latency per element.
    const bool xbulk = n == kBN && ch == kBMaxCh && ((uintptr_t)x & 15) == 0;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        mbar_init(xbar, 1);
        fence_mbar_init();
        for (int s = 0; s < NS && s < l; ++s) issue(s + 1, s);
        if (xbulk) {
            mbar_arrive_expect_tx(xbar, kBN * kBMaxCh * sizeof(float2));
            bulk_g2s(xs, x + (int64_t)g * ch * n, kBN * kBMaxCh * sizeof(float2), xbar);
        }
    }
    // coefficients once into shared memory (the power loop used to re-load them from global)
    for (int idx = tid; idx < H * w; idx += kBTh) {
        const int h = idx / w, t = idx - h * w;
        cs[idx] = (float)coef[(size_t)(g * H + h) * 2 * w + t];
    }
    // X_g (n x ch, column-major) -> xs[c * 64 + j], zero padded
    if (!xbulk)
        for (int idx = tid; idx < kBN * kBMaxCh; idx += kBTh) {
            const int j = idx & 63, c = idx >> 6;
            xs[idx] = (j < n && c < ch) ? x[((int64_t)g * ch + c) * n + j] : make_float2(0.f, 0.f);
        }
    __syncthreads();
    // element ownership: e = tid + 512 u -> i = e & 63 (= tid & 63), j = (tid >> 6) + 8 u
    const int i = tid & 63, j0 = tid >> 6;
    ST q[8][H];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const float c0 = (i == j0 + 8 * u) ? cs[h * w + l] : 0.f;
            if constexpr (R) q[u][h] = c0;
            else q[u][h] = make_float2(c0, 0.f);
        }
    for (int k = 1; k <= l; ++k) {
        const int s = (k - 1) % NS;
        mbar_wait(&full[s], ((k - 1) / NS) & 1);
        const ST* t = regA + (size_t)s * kBSlab;
        float a[H], b[H];
#pragma unroll
        for (int h = 0; h < H; ++h) {
            a[h] = cs[h * w + l + k];
            b[h] = cs[h * w + l - k];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = j0 + 8 * u;
            const ST p = t[bidx(i, j)], pt = t[bidx(j, i)];
#pragma unroll
            for (int h = 0; h < H; ++h) {
                if constexpr (R) {
                    q[u][h] = fmaf(a[h], p, fmaf(b[h], pt, q[u][h]));
                } else {
                    q[u][h].x = fmaf(a[h], p.x, fmaf(b[h], pt.x, q[u][h].x));
                    q[u][h].y = fmaf(a[h], p.y, fmaf(-b[h], pt.y, q[u][h].y));
                }
            }
        }
        __syncthreads();
        if (tid == 0 && k + NS <= l) issue(k + NS, s);
    }
    // Q_h -> region A as column-major 64 x 64: qs[h][j * 64 + i]
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int h = 0; h < H; ++h) regA[(size_t)h * kBN * kBN + (j0 + 8 * u) * kBN + i] = q[u][h];
    if (xbulk) mbar_wait(xbar, 0);
    __syncthreads();
    // Y_h[ii, c] = sum_j Q_h[ii, j] X[j, c]: thread -> rows 2ib, 2ib+1, 32+2ib, 33+2ib and cols 2cb, 2cb+1
    // (the 16 lanes of a half-warp read contiguous bytes of a Q column: conflict-free)
    const int ib = tid & 15, cb = tid >> 4;
    float acc[H][4][2][2];
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c) acc[h][r][c][0] = acc[h][r][c][1] = 0.f;
#pragma unroll 2
    for (int j = 0; j < kBN; ++j) {
        const float2 x0 = xs[(2 * cb) * kBN + j], x1 = xs[(2 * cb + 1) * kBN + j];
#pragma unroll
        for (int h = 0; h < H; ++h) {
            if constexpr (R) {
                const float2* qp = reinterpret_cast<const float2*>(regA + (size_t)h * kBN * kBN + j * kBN + 2 * ib);
                const float2 v0 = qp[0], v1 = qp[16];
                const float qv[4] = {v0.x, v0.y, v1.x, v1.y};
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    acc[h][r][0][0] = fmaf(qv[r], x0.x, acc[h][r][0][0]);
                    acc[h][r][0][1] = fmaf(qv[r], x0.y, acc[h][r][0][1]);
                    acc[h][r][1][0] = fmaf(qv[r], x1.x, acc[h][r][1][0]);
                    acc[h][r][1][1] = fmaf(qv[r], x1.y, acc[h][r][1][1]);
                }
            } else {
                const float4* qp = reinterpret_cast<const float4*>(regA + (size_t)h * kBN * kBN + j * kBN + 2 * ib);
                const float4 v0 = qp[0], v1 = qp[16];
                const float2 qv[4] = {make_float2(v0.x, v0.y), make_float2(v0.z, v0.w), make_float2(v1.x, v1.y),
                                      make_float2(v1.z, v1.w)};
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    acc[h][r][0][0] = fmaf(qv[r].x, x0.x, fmaf(-qv[r].y, x0.y, acc[h][r][0][0]));
                    acc[h][r][0][1] = fmaf(qv[r].x, x0.y, fmaf(qv[r].y, x0.x, acc[h][r][0][1]));
                    acc[h][r][1][0] = fmaf(qv[r].x, x1.x, fmaf(-qv[r].y, x1.y, acc[h][r][1][0]));
                    acc[h][r][1][1] = fmaf(qv[r].x, x1.y, fmaf(qv[r].y, x1.x, acc[h][r][1][1]));
                }
            }
        }
    }
    // y[g][h] : n x ch column-major
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int col = 2 * cb + c;
            if (col >= ch) continue;
            float2* yo = y + (((int64_t)g * H + h) * ch + col) * n;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int row = 2 * ib + (r & 1) + 32 * (r >> 1);
                if (row < n) yo[row] = make_float2(acc[h][r][c][0], acc[h][r][c][1]);
            }
        }
}

constexpr int kBfStages = 4;

// Real-F forward with the Y phase on the tensor cores: Y_h = Q_h X as mma.sync m16n8k8 TF32 with
// the 3xTF32 split (a = a_hi + a_lo, products hi*hi + hi*lo + lo*hi: FP32-level accuracy, far
// inside the complex64 1e-4 bar; single-pass TF32 is not). The FFMA form was issue-bound (FMA pipe
// 51%, 79% of issue slots, profiles/r02_ncu_c5_summary.csv). Shared memory: region Q (the 4-slot
// power ring, then Q_h row-major with a 68-float row stride: conflict-free A fragments), X as
// staged (bulk copy) and its TF32 hi / lo split as the real 64 x 128 matrix [Re | Im interleaved]
// with a 136-float row stride (conflict-free B fragments). One CTA per graph, 16 warps: warp w
// computes m-tile (w & 3) x n-tiles 4 (w >> 2) .. +3 of every head.
constexpr int kBmQs = 68, kBmXs = 136;
constexpr size_t kBmQ = (size_t)kBMaxHeads * kBN * kBmQs * 4;  // 69.6 KB (>= the 64 KB ring)
constexpr size_t kBmXraw = (size_t)kBN * kBMaxCh * 8;           // 32 KB
constexpr size_t kBmXsplit = (size_t)kBN * kBmXs * 4;           // 34.8 KB each (hi, lo)

size_t batch_forward_mma_smem_bytes(int l, int heads) {
    return kBmQ + kBmXraw + 2 * kBmXsplit + (kBfStages + 1) * 8 + (size_t)heads * (2 * l + 1) * 4 + 64;
}

__device__ __forceinline__ uint32_t tf32_of(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return r;
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int H>
__global__ void __launch_bounds__(kBTh, 1)
batch_forward_mma_kernel(const float* __restrict__ slabs, int n, int l, const double* __restrict__ coef,
                         const float2* __restrict__ x, int ch, float2* __restrict__ y) {
    extern __shared__ __align__(128) unsigned char smem[];
    float* regQ = reinterpret_cast<float*>(smem);
    float2* xraw = reinterpret_cast<float2*>(smem + kBmQ);
    float* xhi = reinterpret_cast<float*>(smem + kBmQ + kBmXraw);
    float* xlo = xhi + kBN * kBmXs;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBmQ + kBmXraw + 2 * kBmXsplit);
    uint64_t* xbar = full + kBfStages;
    float* cs = reinterpret_cast<float*>(xbar + 1);
    const int g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int w = 2 * l + 1;
    const float* gs = slabs + (int64_t)g * l * kBSlab;
    constexpr uint32_t bytes = kBSlab * sizeof(float);
    auto issue = [&](int k, int s) {
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(regQ + (size_t)s * kBSlab, gs + (int64_t)(k - 1) * kBSlab, bytes, &full[s]);
    };
    const bool xbulk = n == kBN && ch == kBMaxCh && ((uintptr_t)x & 15) == 0;
    if (tid == 0) {
        for (int s = 0; s < kBfStages; ++s) mbar_init(&full[s], 1);
        mbar_init(xbar, 1);
        fence_mbar_init();
        for (int s = 0; s < kBfStages && s < l; ++s) issue(s + 1, s);
        if (xbulk) {
            mbar_arrive_expect_tx(xbar, kBN * kBMaxCh * sizeof(float2));
            bulk_g2s(xraw, x + (int64_t)g * ch * n, kBN * kBMaxCh * sizeof(float2), xbar);
        }
    }
    for (int idx = tid; idx < H * w; idx += kBTh) {
        const int h = idx / w, t = idx - h * w;
        cs[idx] = (float)coef[(size_t)(g * H + h) * 2 * w + t];
    }
    if (!xbulk)
        for (int idx = tid; idx < kBN * kBMaxCh; idx += kBTh) {
            const int j = idx & 63, c = idx >> 6;
            xraw[idx] = (j < n && c < ch) ? x[((int64_t)g * ch + c) * n + j] : make_float2(0.f, 0.f);
        }
    __syncthreads();
    // power pass: Q_h for 8 elements per thread in registers (both P_ij and P_ji from one staged slab)
    const int i = tid & 63, j0 = tid >> 6;
    float q[8][H];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int h = 0; h < H; ++h) q[u][h] = (i == j0 + 8 * u) ? cs[h * w + l] : 0.f;
    for (int k = 1; k <= l; ++k) {
        const int s = (k - 1) % kBfStages;
        mbar_wait(&full[s], ((k - 1) / kBfStages) & 1);
        const float* t = regQ + (size_t)s * kBSlab;
        float a[H], b[H];
#pragma unroll
        for (int h = 0; h < H; ++h) {
            a[h] = cs[h * w + l + k];
            b[h] = cs[h * w + l - k];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = j0 + 8 * u;
            const float p = t[bidx(i, j)], pt = t[bidx(j, i)];
#pragma unroll
            for (int h = 0; h < H; ++h) q[u][h] = fmaf(a[h], p, fmaf(b[h], pt, q[u][h]));
        }
        __syncthreads();
        if (tid == 0 && k + kBfStages <= l) issue(k + kBfStages, s);
    }
    // Q_h row-major (row i, column j) with stride 68 -- the ring is idle now
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int h = 0; h < H; ++h) regQ[(size_t)h * kBN * kBmQs + i * kBmQs + j0 + 8 * u] = q[u][h];
    if (xbulk) mbar_wait(xbar, 0);
    // X (64 x 64 complex, staged [c][j]) -> the real 64 x 128 matrix Xr[j][2c + e], TF32 hi / lo
    for (int idx = tid; idx < kBN * kBMaxCh; idx += kBTh) {
        const int j = idx & 63, c = idx >> 6;
        const float2 v = xraw[c * kBN + j];
        const float hr = __uint_as_float(tf32_of(v.x)), hm = __uint_as_float(tf32_of(v.y));
        xhi[j * kBmXs + 2 * c] = hr;
        xhi[j * kBmXs + 2 * c + 1] = hm;
        xlo[j * kBmXs + 2 * c] = __uint_as_float(tf32_of(v.x - hr));
        xlo[j * kBmXs + 2 * c + 1] = __uint_as_float(tf32_of(v.y - hm));
    }
    __syncthreads();
    const int gq = lane >> 2, tq = lane & 3;
    const int mt = warp & 3, ng = warp >> 2;
#pragma unroll 1
    for (int h = 0; h < H; ++h) {
        const float* qh = regQ + (size_t)h * kBN * kBmQs;
        float acc[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < kBN / 8; ++ks) {
            // A fragment: a0 = Q[16mt + g][8ks + t], a1 = row + 8, a2 = column + 4, a3 = both
            const float* qa = qh + (16 * mt + gq) * kBmQs + 8 * ks + tq;
            const float av[4] = {qa[0], qa[8 * kBmQs], qa[4], qa[8 * kBmQs + 4]};
            uint32_t ahi[4], alo[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                ahi[e] = tf32_of(av[e]);
                alo[e] = tf32_of(av[e] - __uint_as_float(ahi[e]));
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                // B fragment: b0 = Xr[8ks + t][8(4ng + nt) + g], b1 = row + 4
                const int col = 8 * (4 * ng + nt) + gq, row = 8 * ks + tq;
                const uint32_t bh0 = __float_as_uint(xhi[row * kBmXs + col]);
                const uint32_t bh1 = __float_as_uint(xhi[(row + 4) * kBmXs + col]);
                const uint32_t bl0 = __float_as_uint(xlo[row * kBmXs + col]);
                const uint32_t bl1 = __float_as_uint(xlo[(row + 4) * kBmXs + col]);
                mma_tf32(acc[nt], alo, bh0, bh1);  // small terms first
                mma_tf32(acc[nt], ahi, bl0, bl1);
                mma_tf32(acc[nt], ahi, bh0, bh1);
            }
        }
        // D fragment: (c0, c1) = Y_h[16mt + g][real cols 2t, 2t+1 of n-tile] = one complex value,
        // (c2, c3) the same for row + 8
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            const int cc = 4 * (4 * ng + nt) + tq;  // complex column
            if (cc >= ch) continue;
            float2* yo = y + (((int64_t)g * H + h) * ch + cc) * n;
            const int r0 = 16 * mt + gq;
            if (r0 < n) yo[r0] = make_float2(acc[nt][0], acc[nt][1]);
            if (r0 + 8 < n) yo[r0 + 8] = make_float2(acc[nt][2], acc[nt][3]);
        }
    }
}

template <int H, bool R>
__global__ void __launch_bounds__(kBTh, 1)
batch_dlda_kernel(const void* __restrict__ slabs, int n, int l, const double* __restrict__ coef,
                  const float2* __restrict__ gcot, const float2* __restrict__ x, int ch, double* __restrict__ dlda) {
    using ST = typename std::conditional<R, float, float2>::type;  // slab element; M element (Re M for R)
    extern __shared__ __align__(128) unsigned char smem[];
    float2* regA = reinterpret_cast<float2*>(smem);
    ST* regS = reinterpret_cast<ST*>(smem);  // the same region as power stages
    float2* xs = reinterpret_cast<float2*>(smem + BatchSmem::kA);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + BatchSmem::kA + BatchSmem::kX);
    uint64_t* xbar = full + kBStagesR;
    double* red = reinterpret_cast<double*>(xbar + 1);  // [k 0..l][warp 16][8]
    const int g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int w = 2 * l + 1;
    const ST* gs = static_cast<const ST*>(slabs) + (int64_t)g * l * kBSlab;
    // full-size graphs: X_g and the H gradient blocks G_h are contiguous in the staged layouts, so
    // two bulk copies replace the per-element loads
    const bool bulk = n == kBN && ch == kBMaxCh && ((uintptr_t)x & 15) == 0 && ((uintptr_t)gcot & 15) == 0;
    if (tid == 0) {
        for (int s = 0; s < kBStages; ++s) mbar_init(&full[s], 1);
        mbar_init(xbar, 1);
        fence_mbar_init();
        if (bulk) {
            constexpr uint32_t blk = kBN * kBMaxCh * sizeof(float2);
            mbar_arrive_expect_tx(xbar, (H + 1) * blk);
            bulk_g2s(xs, x + (int64_t)g * ch * n, blk, xbar);
            bulk_g2s(regA, gcot + (int64_t)g * H * ch * n, H * blk, xbar);
        }
    }
    // stage X (xs[c*64 + j]) and G_h (regA[h][c*64 + i]), zero padded
    if (!bulk)
        for (int idx = tid; idx < kBN * kBMaxCh; idx += kBTh) {
            const int r = idx & 63, c = idx >> 6;
            const bool v = r < n && c < ch;
            xs[idx] = v ? x[((int64_t)g * ch + c) * n + r] : make_float2(0.f, 0.f);
#pragma unroll
            for (int h = 0; h < H; ++h)
                regA[(size_t)h * kBN * kBMaxCh + idx] =
                    v ? gcot[(((int64_t)g * H + h) * ch + c) * n + r] : make_float2(0.f, 0.f);
        }
    __syncthreads();
    if (bulk) mbar_wait(xbar, 0);
    // M_h[i, j] = sum_c G_h[i, c] conj(X[j, c]) for the thread's 8 elements
    const int i = tid & 63, j0 = tid >> 6;
    ST m[8][H];  // R: only Re M = Gr Xr^T + Gi Xi^T is needed against real powers
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int h = 0; h < H; ++h) {
            if constexpr (R) m[u][h] = 0.f;
            else m[u][h] = make_float2(0.f, 0.f);
        }
    for (int c = 0; c < kBMaxCh; ++c) {
        float2 gv[H];
#pragma unroll
        for (int h = 0; h < H; ++h) gv[h] = regA[(size_t)h * kBN * kBMaxCh + c * kBN + i];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const float2 xv = xs[c * kBN + j0 + 8 * u];
#pragma unroll
            for (int h = 0; h < H; ++h) {  // g * conj(x)
                if constexpr (R) {
                    m[u][h] = fmaf(gv[h].x, xv.x, fmaf(gv[h].y, xv.y, m[u][h]));
                } else {
                    m[u][h].x = fmaf(gv[h].x, xv.x, fmaf(gv[h].y, xv.y, m[u][h].x));
                    m[u][h].y = fmaf(gv[h].y, xv.x, fmaf(-gv[h].x, xv.y, m[u][h].y));
                }
            }
        }
    }
    __syncthreads();  // region A is reused for the power stages
    const uint32_t bytes = kBSlab * sizeof(ST);
    auto issue = [&](int k, int s) {
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(regS + (size_t)s * kBSlab, gs + (int64_t)(k - 1) * kBSlab, bytes, &full[s]);
    };
    if (tid == 0)
        for (int s = 0; s < kBStages && s < l; ++s) issue(s + 1, s);
    // s_0 = Re tr(M_h)
    {
        double v[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) v[h] = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int h = 0; h < H; ++h)
                if (i == j0 + 8 * u) {
                    if constexpr (R) v[h] += (double)m[u][h];
                    else v[h] += (double)m[u][h].x;
                }
#pragma unroll
        for (int h = 0; h < H; ++h) {
            double t = v[h];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (lane == 0) red[(0 * 16 + warp) * 8 + h] = t;
        }
    }
    for (int k = 1; k <= l; ++k) {
        const int s = (k - 1) % kBStages;
        mbar_wait(&full[s], ((k - 1) / kBStages) & 1);
        const ST* t = regS + (size_t)s * kBSlab;
        // [h][+/-] packed as 2h + sign; the thread's 8 terms are summed in FP32 (one F2F per value
        // instead of one per product), the cross-thread reduction is FP64
        float vf[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) vf[q] = 0.f;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = j0 + 8 * u;
            const ST p = t[bidx(i, j)], pt = t[bidx(j, i)];
#pragma unroll
            for (int h = 0; h < H; ++h) {
                if constexpr (R) {
                    vf[2 * h] = fmaf(m[u][h], p, vf[2 * h]);
                    vf[2 * h + 1] = fmaf(m[u][h], pt, vf[2 * h + 1]);
                } else {
                    vf[2 * h] += fmaf(m[u][h].x, p.x, m[u][h].y * p.y);
                    vf[2 * h + 1] += fmaf(m[u][h].x, pt.x, -m[u][h].y * pt.y);
                }
            }
        }
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = (double)vf[q];
        // transposing warp reduction of 8 values: lane q (< 8) ends with the sum of value q
#pragma unroll
        for (int o = 4, half = 4; o >= 1; o >>= 1, half >>= 1) {
            const bool hi = (lane & o) != 0;
#pragma unroll
            for (int q = 0; q < half; ++q) {
                const double send = hi ? v[q] : v[q + half];
                const double keep = hi ? v[q + half] : v[q];
                v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 8);
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 16);
        if (lane < 8) red[(k * 16 + warp) * 8 + lane] = v[0];
        __syncthreads();
        if (tid == 0 && k + kBStages <= l) issue(k + kBStages, s);
    }
    __syncthreads();
    // per-power totals over the 16 warps, one thread per (power, value), in place in warp 0's row
    // (only this thread touches its column); then dL/da_h = sum_k c'_k s_hk by H threads
    for (int t = tid; t < (l + 1) * 8; t += kBTh) {
        const int kr = t >> 3, q = t & 7;
        double sk = 0.0;
#pragma unroll
        for (int wp = 0; wp < 16; ++wp) sk += red[(kr * 16 + wp) * 8 + q];
        red[(kr * 16) * 8 + q] = sk;
    }
    __syncthreads();
    if (tid < H) {
        const int h = tid;
        const double* dc = coef + (size_t)(g * H + h) * 2 * w + w;
        double acc = 0.0;
        for (int kk = 0; kk < w; ++kk) {  // ascending k = -l..l
            const int k = kk - l;
            const int kr = k >= 0 ? k : -k;
            acc += dc[kk] * red[(kr * 16) * 8 + (k == 0 ? h : (k > 0 ? 2 * h : 2 * h + 1))];
        }
        dlda[(int64_t)g * H + h] = acc;
    }
}

// ---------------------------------------------------------------- config 5 on the tensor cores
//
// Real F, n = 64, 64 channels (the BASELINE config-5 shape): persistent, warp-specialised kernels,
// one CTA per SM walking graphs g = blockIdx.x, + gridDim.x, ... Warp 16 streams every 16 KB item
// a graph needs (its real power slabs, X_g in two channel halves, and for dL/da the gradient blocks
// G_h) through ONE ring of bulk copies that runs ahead ACROSS graphs, so HBM never waits for a
// graph's compute; warp 17 issues the graph's GEMM on tcgen05 (kind::f16, BF16 operands, FP32
// accumulators in TMEM); warps 0..15 synthesise Q_h from the powers in registers (thread = element
// (i, 8 jb .. 8 jb + 7), all heads: each staged power value is read once for every head), write the
// GEMM operands and drain TMEM. FP32-level accuracy from BF16 operands by the two-term split
// a = a_hi + a_lo (products hi hi + hi lo + lo hi: ~2^-16 relative, inside the complex64 1e-4 bar;
// the 2^-32 term is dropped). Operands are K-major SWIZZLE_NONE canonical layouts with 64-byte K
// blocks: byte(r, k) = (k / 32) rows 64 + (r / 8) 512 + ((k % 32) / 8) 128 + (r % 8) 16 + (k % 8) 2.
//   forward: [Y_h0; Y_h1] (128 x 128 real: columns 2c + re/im) = [Q_h0; Q_h1] (128 x 64) X^T (64 x 128)
//   dL/da:   [M_h0; M_h1] (128 x 64) = [G_h0; G_h1] (128 x 128: K = 2c + re/im) [X] (64 x 128),
//            Re M_h = Re(G_h X^H); s_hk = <M_h, P_k>, <M_h, P_k^T> and dL/da_h = sum_k c'_k s_hk.
constexpr int kTcItem = kBSlab * 4;           // 16 KB: a real power slab / half of X_g / half of G_h
constexpr int kTcWarps = 16;                  // synthesis / operand / epilogue warps
constexpr int kTcThreads = 32 * (kTcWarps + 2);
constexpr int kTcMaxStages = 8;

// byte offset of the 16-byte chunk (row r, K core column k8 = k / 8) of a rows x K canonical operand
__device__ __forceinline__ uint32_t tc_off(int rows, int r, int k8) {
    return (uint32_t)((k8 >> 2) * rows * 64 + (r >> 3) * 512 + (k8 & 3) * 128 + (r & 7) * 16);
}

// 8 floats -> BF16 hi / lo chunks (a = hi + lo + O(2^-17 a))
__device__ __forceinline__ void tc_split8(const float (&v)[8], uint4& hi, uint4& lo) {
    uint32_t h[4], l[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const __nv_bfloat162 bh = __floats2bfloat162_rn(v[2 * q], v[2 * q + 1]);
        const float2 back = __bfloat1622float2(bh);
        const __nv_bfloat162 bl = __floats2bfloat162_rn(v[2 * q] - back.x, v[2 * q + 1] - back.y);
        h[q] = *reinterpret_cast<const uint32_t*>(&bh);
        l[q] = *reinterpret_cast<const uint32_t*>(&bl);
    }
    hi = make_uint4(h[0], h[1], h[2], h[3]);
    lo = make_uint4(l[0], l[1], l[2], l[3]);
}

__device__ __forceinline__ void st_shared_v4(unsigned char* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }

__device__ __forceinline__ void tc_compute_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kTcWarps) : "memory"); }

// Ring position: stage and phase parity advanced item by item (no division in the loops). The
// producer waits on `empty` with the opposite parity, which a fresh barrier passes at once.
struct TcCursor {
    int s = 0;
    uint32_t ph = 0;
    __device__ __forceinline__ void next(int stages) {
        if (++s == stages) {
            s = 0;
            ph ^= 1u;
        }
    }
};

struct TcRing {
    unsigned char* base;
    uint64_t* full;
    uint64_t* empty;
    int stages;
    __device__ __forceinline__ const unsigned char* wait(const TcCursor& c) const {
        mbar_wait(full + c.s, c.ph);
        return base + (size_t)c.s * kTcItem;
    }
    __device__ __forceinline__ void release(const TcCursor& c, int lane) const {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + c.s);
    }
    __device__ __forceinline__ void produce(TcCursor& c, const void* src, uint64_t pol) const {
        mbar_wait(empty + c.s, c.ph ^ 1u);
        mbar_arrive_expect_tx(full + c.s, kTcItem);
        bulk_g2s_hint(base + (size_t)c.s * kTcItem, src, kTcItem, full + c.s, pol);
        c.next(stages);
    }
};

// Per-graph series coefficients, FP32 (batch_coef_kernel's second table): [h][c | c'][2l + 1] at a
// per-graph stride padded to 16 bytes, double-buffered in shared memory by graph parity and
// bulk-copied by the producer ahead of the graph's first ring item (no CTA barrier per graph).
__host__ __device__ constexpr int tc_coef_stride(int heads, int l) { return 16 * (l + 1) + 0 * heads; }

struct TcCoefs {
    float* buf;      // [2][stride]
    uint64_t* full;  // [2]
    uint64_t* empty; // [2], one arrival per compute warp
    int stride;
    __device__ __forceinline__ const float* wait(int t) const {
        mbar_wait(full + (t & 1), (uint32_t)((t >> 1) & 1));
        return buf + (t & 1) * stride;
    }
    __device__ __forceinline__ void release(int t, int lane) const {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + (t & 1));
    }
    __device__ __forceinline__ void produce(int t, const float* src) const {
        mbar_wait(empty + (t & 1), (uint32_t)(((t >> 1) & 1) ^ 1));
        mbar_arrive_expect_tx(full + (t & 1), (uint32_t)stride * 4);
        bulk_g2s(buf + (t & 1) * stride, src, (uint32_t)stride * 4, full + (t & 1));
    }
};

// the coefficient buffers are bulk-copy destinations: 16-byte aligned
__device__ __forceinline__ float* tc_align16(void* p) {
    return reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(p) + 15) & ~(uintptr_t)15);
}

// barriers: full[8], empty[8], cfull[2], cempty[2], opready, mmadone, tempty; then the TMEM slot
constexpr int kTcBars = 2 * kTcMaxStages + 4 + 3;

__device__ __forceinline__ void tc_init_barriers(uint64_t* bars, int stages, int op_count) {
    for (int s = 0; s < stages; ++s) {
        mbar_init(bars + s, 1);
        mbar_init(bars + kTcMaxStages + s, kTcWarps);
    }
    uint64_t* c = bars + 2 * kTcMaxStages;
    mbar_init(c + 0, 1);
    mbar_init(c + 1, 1);
    mbar_init(c + 2, kTcWarps);
    mbar_init(c + 3, kTcWarps);
    mbar_init(c + 4, op_count);  // opready
    mbar_init(c + 5, 1);         // mmadone
    mbar_init(c + 6, kTcWarps);  // tempty (unused by the current kernels' single TMEM buffer)
    fence_mbar_init();
}

// ring depth cap (FGFRFT_TC_STAGES: experiments only)
static int tc_max_stages() {
    static const int v = [] {
        const char* e = std::getenv("FGFRFT_TC_STAGES");
        const int s = e ? std::atoi(e) : kTcMaxStages;
        return s >= 3 && s <= kTcMaxStages ? s : kTcMaxStages;
    }();
    return v;
}

size_t batch_tc_fwd_smem(int l, int heads, int* stages) {
    const size_t ops = (size_t)((heads + 1) / 2) * 2 * 16384 + 2 * 16384;  // Q tiles hi / lo, X^T hi / lo
    const size_t fixed = ops + kTcBars * 8 + 16 + 2 * (size_t)tc_coef_stride(heads, l) * 4 + 128;
    int st = (int)((227 * 1024 - fixed) / kTcItem);
    if (st > tc_max_stages()) st = tc_max_stages();
    if (stages) *stages = st;
    return fixed + (size_t)st * kTcItem;
}

// Forward. The compute warps run graph t's epilogue AFTER synthesising graph t + 1 (the MMA of t
// overlaps that synthesis), then write t + 1's operands: operands and TMEM stay single-buffered
// because graph t's accumulators are drained before t + 1's MMA is released.
template <int H>
__global__ void __launch_bounds__(kTcThreads, 1)
batch_fwd_tc_kernel(const float* __restrict__ slabs, int l, const float* __restrict__ coef,
                    const float2* __restrict__ x, float2* __restrict__ y, int graphs, int stages) {
    constexpr int NT = (H + 1) / 2;  // M tiles of two heads
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* qhl = smem;                        // [NT][hi, lo] 128 x 64 BF16 (16 KB each)
    unsigned char* xhl = qhl + NT * 2 * 16384;        // [hi, lo] X^T: 128 x 64 BF16
    unsigned char* ringp = xhl + 2 * 16384;
    uint64_t* bars = reinterpret_cast<uint64_t*>(ringp + (size_t)stages * kTcItem);
    const TcRing ring{ringp, bars, bars + kTcMaxStages, stages};
    uint64_t* opready = bars + 2 * kTcMaxStages + 4;
    uint64_t* mmadone = opready + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + kTcBars);
    const int cst = tc_coef_stride(H, l);
    const TcCoefs cf{tc_align16(tslot + 4), bars + 2 * kTcMaxStages, bars + 2 * kTcMaxStages + 2, cst};
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) tc_init_barriers(bars, stages, kTcWarps);
    if (warp == kTcWarps + 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    if (warp == kTcWarps) {
        // ---- producer: per graph its coefficients, the l power slabs, then X_g (channels 0-31, 32-63)
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            TcCursor c;
            int t = 0;
            for (int g = blockIdx.x; g < graphs; g += gridDim.x, ++t) {
                cf.produce(t, coef + (size_t)g * cst);
                for (int k = 0; k < l; ++k) ring.produce(c, slabs + ((int64_t)g * l + k) * kBSlab, pol);
                for (int hh = 0; hh < 2; ++hh)
                    ring.produce(c, x + (int64_t)g * kBN * kBMaxCh + hh * (kBN * kBMaxCh / 2), pol);
            }
        }
    } else if (warp == kTcWarps + 1) {
        // ---- MMA issuer: per graph NT tiles x 4 K steps x 3 split products
        if (lane == 0) {
            const uint32_t q0 = smem_u32(qhl), x0 = smem_u32(xhl);
            int t = 0;
            for (int g = blockIdx.x; g < graphs; g += gridDim.x, ++t) {
                mbar_wait(opready, (uint32_t)(t & 1));
                tc_fence_after();
#pragma unroll
                for (int mt = 0; mt < NT; ++mt)
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
#pragma unroll
                        for (int ps = 0; ps < 3; ++ps) {  // lo hi, hi lo, hi hi (small terms first)
                            const uint32_t a = q0 + (uint32_t)(mt * 2 + (ps == 0)) * 16384u;
                            const uint32_t b = x0 + (uint32_t)(ps == 1) * 16384u;
                            const uint32_t ko = (uint32_t)((ks >> 1) * 8192 + (ks & 1) * 256);
                            mma_bf16(tmem + (uint32_t)(mt * 128), umma_desc(a + ko, 128, 512),
                                     umma_desc(b + ko, 128, 512), idesc_bf16(128, 128), (ks | ps) ? 1u : 0u);
                        }
                mma_commit(mmadone);
            }
        }
    } else {
        // ---- compute warps
        const int tid = threadIdx.x, i = tid & 63, jb = tid >> 6;
        const int qd = warp & 3, wq = warp >> 2;  // TMEM lane quarter, column quarter
        // graph pg's Y from TMEM: lane 32 qd + lane of tile mt = row (h, i); this warp's 32 columns
        auto epilogue = [&](int pg) {
#pragma unroll
            for (int mt = 0; mt < NT; ++mt) {
                const int h = 2 * mt + (qd >> 1), io = 32 * (qd & 1) + lane;
                if (h >= H) continue;  // warp-uniform
                float2* yo = y + (((int64_t)pg * H + h) * kBMaxCh + 16 * wq) * kBN + io;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {  // 16 columns at a time: the next graph's Q is live
                    int32_t v[16];
                    tmem_ld16(tmem + ((uint32_t)(32 * qd) << 16) + (uint32_t)(mt * 128 + 32 * wq + 16 * hf), v);
                    tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        __stcs(yo + (8 * hf + c) * kBN,
                               make_float2(__int_as_float(v[2 * c]), __int_as_float(v[2 * c + 1])));
                }
            }
        };
        TcCursor rc;
        int t = 0, pg = -1;
        for (int g = blockIdx.x; g < graphs; g += gridDim.x, ++t) {
            const float4* cs = reinterpret_cast<const float4*>(cf.wait(t));  // [c_k | c_-k][k][4 heads]
            float q[H][8];
            {
                const float4 c0 = cs[0];
                const float c0v[4] = {c0.x, c0.y, c0.z, c0.w};
#pragma unroll
                for (int h = 0; h < H; ++h)
#pragma unroll
                    for (int u = 0; u < 8; ++u) q[h][u] = (i == 8 * jb + u) ? c0v[h] : 0.f;
            }
            for (int k = 1; k <= l; ++k) {
                const float* tp = reinterpret_cast<const float*>(ring.wait(rc));
                const float4 av = cs[k], bv = cs[l + 1 + k];
                const float a[4] = {av.x, av.y, av.z, av.w}, b[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int j = 8 * jb + u;
                    const float p = tp[bidx(i, j)], pt = tp[bidx(j, i)];
#pragma unroll
                    for (int h = 0; h < H; ++h) q[h][u] = fmaf(a[h], p, fmaf(b[h], pt, q[h][u]));
                }
                ring.release(rc, lane);
                rc.next(stages);
            }
            cf.release(t, lane);
            // the previous graph's MMA ran during this synthesis: once it is done, Q moves into the
            // operand tiles (so the accumulators are not live during the epilogue), the previous
            // graph's Y leaves TMEM, and X_g takes the operand the MMA has finished reading
            if (pg >= 0) mbar_wait(mmadone, (uint32_t)((t - 1) & 1));
            // Q_h -> A operand of tile h / 2: row (h % 2) 64 + i, K core column jb
#pragma unroll
            for (int h = 0; h < H; ++h) {
                uint4 hi, lo;
                tc_split8(q[h], hi, lo);
                unsigned char* tq = qhl + (size_t)(h >> 1) * 2 * 16384;
                st_shared_v4(tq + tc_off(128, (h & 1) * 64 + i, jb), hi);
                st_shared_v4(tq + 16384 + tc_off(128, (h & 1) * 64 + i, jb), lo);
            }
            if (pg >= 0) {
                tc_fence_after();
                epilogue(pg);
                tc_fence_before();
            }
            // X_g halves -> X^T operand: B row n = 2c + e, K = j. Thread: channel c = 32 half + cl
            // (cl = tid >> 3 & 31), 8 consecutive j (kc = tid & 7), both components -> rows 2c, 2c + 1.
            {
                const int half = tid >> 8, cl = (tid >> 3) & 31, kc = tid & 7;
                for (int hh = 0; hh < 2; ++hh) {
                    const float2* xr = reinterpret_cast<const float2*>(ring.wait(rc));
                    if (hh == half) {
                        // chunk (m + kc / 2) % 4 first: the 8 lanes of a channel then hit 8 distinct
                        // 16-byte bank groups (kc * 64 bytes alone covers only two)
                        const int rot = kc >> 1;
                        float4 ld[4];
#pragma unroll
                        for (int m = 0; m < 4; ++m)
                            ld[m] = *reinterpret_cast<const float4*>(xr + cl * kBN + 8 * kc + 2 * ((m + rot) & 3));
                        float re[8], im[8];
#pragma unroll
                        for (int m = 0; m < 4; ++m) {  // chunk m was loaded as ld[(m - rot) & 3]
                            const float4 v = rot == 0 ? ld[m] : rot == 1 ? ld[(m + 3) & 3] : rot == 2 ? ld[(m + 2) & 3] : ld[(m + 1) & 3];
                            re[2 * m] = v.x;
                            im[2 * m] = v.y;
                            re[2 * m + 1] = v.z;
                            im[2 * m + 1] = v.w;
                        }
                        const int n0 = 2 * (32 * half + cl);
                        uint4 rh, rl, ih, il;
                        tc_split8(re, rh, rl);
                        tc_split8(im, ih, il);
                        // odd kc lanes store their imaginary row first: each store instruction then
                        // covers all 8 16-byte bank groups of a 128-byte row group (2x fewer wavefronts)
                        const int sw = kc & 1, na = n0 + sw, nb = n0 + 1 - sw;
                        st_shared_v4(xhl + tc_off(128, na, kc), sw ? ih : rh);
                        st_shared_v4(xhl + 16384 + tc_off(128, na, kc), sw ? il : rl);
                        st_shared_v4(xhl + tc_off(128, nb, kc), sw ? rh : ih);
                        st_shared_v4(xhl + 16384 + tc_off(128, nb, kc), sw ? rl : il);
                    }
                    ring.release(rc, lane);
                    rc.next(stages);
                }
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(opready);
            pg = g;
        }
        if (pg >= 0) {
            mbar_wait(mmadone, (uint32_t)((t - 1) & 1));
            tc_fence_after();
            epilogue(pg);
            tc_fence_before();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kTcWarps + 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

constexpr int kTcMs = 68;  // row stride (floats) of the staged M_h: conflict-free row-chunk reads

size_t batch_tc_dlda_smem(int l, int heads, int* stages) {
    const size_t mreg = (size_t)kBMaxHeads * kBN * kTcMs * 4;  // >= one G tile hi / lo (64 KB)
    const size_t fixed = 2 * 16384 + mreg + kTcBars * 8 + 16 + 2 * (size_t)tc_coef_stride(heads, l) * 4 +
                         kTcWarps * kBMaxHeads * 8 + 128;
    int st = (int)((227 * 1024 - fixed) / kTcItem);
    if (st > tc_max_stages()) st = tc_max_stages();
    if (stages) *stages = st;
    return fixed + (size_t)st * kTcItem;
}

template <int H>
__global__ void __launch_bounds__(kTcThreads, 1)
batch_dlda_tc_kernel(const float* __restrict__ slabs, int l, const float* __restrict__ coef,
                     const float2* __restrict__ gcot, const float2* __restrict__ x, double* __restrict__ dlda,
                     int graphs, int stages) {
    constexpr int NT = (H + 1) / 2;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* xhl = smem;                 // [hi, lo] X: 64 rows (j) x 128 K (2c + e) BF16 (16 KB each)
    unsigned char* reg = xhl + 2 * 16384;      // G tile [hi, lo] 128 x 128 BF16, later M_h [h][i][kTcMs]
    float* ms = reinterpret_cast<float*>(reg);
    unsigned char* ringp = reg + (size_t)kBMaxHeads * kBN * kTcMs * 4;
    uint64_t* bars = reinterpret_cast<uint64_t*>(ringp + (size_t)stages * kTcItem);
    const TcRing ring{ringp, bars, bars + kTcMaxStages, stages};
    uint64_t* opready = bars + 2 * kTcMaxStages + 4;
    uint64_t* mmadone = opready + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + kTcBars);
    const int cst = tc_coef_stride(H, l);
    const TcCoefs cf{tc_align16(tslot + 4), bars + 2 * kTcMaxStages, bars + 2 * kTcMaxStages + 2, cst};
    double* red = reinterpret_cast<double*>(cf.buf + 2 * cst);  // [16 warps][4]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) tc_init_barriers(bars, stages, kTcWarps);
    if (warp == kTcWarps + 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    constexpr int kHalf = kBN * kBMaxCh / 2;  // float2 elements of half a 64 x 64 complex block
    if (warp == kTcWarps) {
        // ---- producer: per graph its coefficients, X_g (2 items), G_h (2 items per head), the powers
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            TcCursor c;
            int t = 0;
            for (int g = blockIdx.x; g < graphs; g += gridDim.x, ++t) {
                cf.produce(t, coef + (size_t)g * cst);
                for (int hh = 0; hh < 2; ++hh) ring.produce(c, x + (int64_t)g * kBN * kBMaxCh + hh * kHalf, pol);
                for (int hh = 0; hh < 2 * H; ++hh)
                    ring.produce(c, gcot + (int64_t)g * H * kBN * kBMaxCh + hh * kHalf, pol);
                for (int k = 0; k < l; ++k) ring.produce(c, slabs + ((int64_t)g * l + k) * kBSlab, pol);
            }
        }
    } else if (warp == kTcWarps + 1) {
        // ---- MMA issuer: per graph NT tiles, each 8 K steps x 3 split products (N = 64)
        if (lane == 0) {
            const uint32_t x0 = smem_u32(xhl), a0 = smem_u32(reg);
            int ev = 0;
            for (int g = blockIdx.x; g < graphs; g += gridDim.x)
                for (int mt = 0; mt < NT; ++mt, ++ev) {
                    mbar_wait(opready, (uint32_t)(ev & 1));
                    tc_fence_after();
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks)
#pragma unroll
                        for (int ps = 0; ps < 3; ++ps) {
                            const uint32_t a = a0 + (uint32_t)(ps == 0) * 32768u + (uint32_t)((ks >> 1) * 8192 + (ks & 1) * 256);
                            const uint32_t b = x0 + (uint32_t)(ps == 1) * 16384u + (uint32_t)((ks >> 1) * 4096 + (ks & 1) * 256);
                            mma_bf16(tmem + (uint32_t)(mt * 64), umma_desc(a, 128, 512), umma_desc(b, 128, 512),
                                     idesc_bf16(128, 64), (ks | ps) ? 1u : 0u);
                        }
                    mma_commit(mmadone);
                }
        }
    } else {
        const int tid = threadIdx.x, i = tid & 63, jb = tid >> 6;
        const int qd = warp & 3, wq = warp >> 2;
        TcCursor rc;
        int t = 0, ev = 0;
        // one 16 KB half (channels 32 hh ..) of a complex 64 x 64 block -> 8 values of operand row r
        // (K core column 8 hh + jb: channels 4 jb .. 4 jb + 3 of the half, re / im interleaved)
        auto convert = [&](unsigned char* dst, int rows, int r, int hh, uint32_t lo_off) {
            const float2* src = reinterpret_cast<const float2*>(ring.wait(rc));
            float v[8];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const float2 z = src[(4 * jb + m) * kBN + i];
                v[2 * m] = z.x;
                v[2 * m + 1] = z.y;
            }
            uint4 hi, lo;
            tc_split8(v, hi, lo);
            st_shared_v4(dst + tc_off(rows, r, 8 * hh + jb), hi);
            st_shared_v4(dst + lo_off + tc_off(rows, r, 8 * hh + jb), lo);
            ring.release(rc, lane);
            rc.next(stages);
        };
        for (int g = blockIdx.x; g < graphs; g += gridDim.x, ++t) {
            for (int hh = 0; hh < 2; ++hh) convert(xhl, 64, i, hh, 16384);
            for (int mt = 0; mt < NT; ++mt, ++ev) {
                if (mt > 0) mbar_wait(mmadone, (uint32_t)((ev - 1) & 1));  // tile mt - 1 has read the region
                for (int hl = 0; hl < 2; ++hl) {
                    if (2 * mt + hl >= H) break;
                    for (int hh = 0; hh < 2; ++hh) convert(reg, 128, 64 * hl + i, hh, 32768);
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(opready);
            }
            mbar_wait(mmadone, (uint32_t)((ev - 1) & 1));
            tc_fence_after();
            // M_h rows (TMEM lane 32 qd + lane of tile mt) -> ms[h][i][j], this warp's 16 columns
#pragma unroll
            for (int mt = 0; mt < NT; ++mt) {
                const int h = 2 * mt + (qd >> 1), io = 32 * (qd & 1) + lane;
                if (h >= H) continue;
                int32_t v[16];
                tmem_ld16(tmem + ((uint32_t)(32 * qd) << 16) + (uint32_t)(mt * 64 + 16 * wq), v);
                tmem_wait_ld();
                float4* dst = reinterpret_cast<float4*>(ms + ((size_t)h * kBN + io) * kTcMs + 16 * wq);
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    dst[c] = make_float4(__int_as_float(v[4 * c]), __int_as_float(v[4 * c + 1]),
                                         __int_as_float(v[4 * c + 2]), __int_as_float(v[4 * c + 3]));
            }
            tc_fence_before();
            tc_compute_sync();
            float m[H][8];
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const float4* src = reinterpret_cast<const float4*>(ms + ((size_t)h * kBN + i) * kTcMs + 8 * jb);
                const float4 a = src[0], b = src[1];
                m[h][0] = a.x; m[h][1] = a.y; m[h][2] = a.z; m[h][3] = a.w;
                m[h][4] = b.x; m[h][5] = b.y; m[h][6] = b.z; m[h][7] = b.w;
            }
            tc_compute_sync();  // the region is the next graph's G tile
            const float4* dcs = reinterpret_cast<const float4*>(cf.wait(t)) + 2 * (l + 1);  // [c'_k | c'_-k][k][4]
            float dl[H];
            {
                const float4 d0 = dcs[0];
                const float d0v[4] = {d0.x, d0.y, d0.z, d0.w};
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    float d = 0.f;
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (i == 8 * jb + u) d = m[h][u];
                    dl[h] = d0v[h] * d;  // c'_0 Re tr(M_h)
                }
            }
            for (int k = 1; k <= l; ++k) {
                const float* tp = reinterpret_cast<const float*>(ring.wait(rc));
                float vp[H], vm[H];
#pragma unroll
                for (int h = 0; h < H; ++h) vp[h] = vm[h] = 0.f;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int j = 8 * jb + u;
                    const float p = tp[bidx(i, j)], pt = tp[bidx(j, i)];
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                        vp[h] = fmaf(m[h][u], p, vp[h]);
                        vm[h] = fmaf(m[h][u], pt, vm[h]);
                    }
                }
                ring.release(rc, lane);
                rc.next(stages);
                const float4 dpv = dcs[k], dmv = dcs[l + 1 + k];
                const float dp[4] = {dpv.x, dpv.y, dpv.z, dpv.w}, dm[4] = {dmv.x, dmv.y, dmv.z, dmv.w};
#pragma unroll
                for (int h = 0; h < H; ++h) dl[h] = fmaf(dp[h], vp[h], fmaf(dm[h], vm[h], dl[h]));
            }
            cf.release(t, lane);
            // FP32 per thread (8 elements x 2l + 1 terms), FP64 across the 512 threads
#pragma unroll
            for (int h = 0; h < H; ++h) {
                double s2 = (double)dl[h];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
                if (lane == 0) red[warp * kBMaxHeads + h] = s2;
            }
            tc_compute_sync();
            if (tid < H) {
                double s2 = 0.0;
                for (int wp = 0; wp < kTcWarps; ++wp) s2 += red[wp * kBMaxHeads + tid];
                dlda[(int64_t)g * H + tid] = s2;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kTcWarps + 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// The tcgen05 kernels' shape: full 64-node graphs, 64 channels, 16-byte aligned signal blocks.
static bool tc_shape_ok(int n, int ch, const void* a, const void* b) {
    return n == kBN && ch == kBMaxCh && ((uintptr_t)a & 15) == 0 && ((uintptr_t)b & 15) == 0;
}

static size_t batch_coef_dbytes(int n_orders, int l) { return ((size_t)n_orders * 2 * (2 * l + 1) * 8 + 15) & ~(size_t)15; }

size_t batch_coef_bytes(int graphs, int heads, int l) {
    return batch_coef_dbytes(graphs * heads, l) + (size_t)graphs * tc_coef_stride(heads, l) * 4;
}

static const float* batch_coef_f(const double* coef, int n_orders, int l) {
    return reinterpret_cast<const float*>(reinterpret_cast<const char*>(coef) + batch_coef_dbytes(n_orders, l));
}

cudaError_t launch_batch_coef(const double* alphas_dev, int n_orders, int l, double* coef_dev, cudaStream_t stream,
                              int heads) {
    const int total = n_orders * (2 * l + 1);
    float* cf = heads > 0 ? const_cast<float*>(batch_coef_f(coef_dev, n_orders, l)) : nullptr;
    batch_coef_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, stream>>>(alphas_dev, n_orders, l, coef_dev, cf,
                                                                          heads > 0 ? heads : 1,
                                                                          tc_coef_stride(heads > 0 ? heads : 1, l));
    return cudaGetLastError();
}

cudaError_t launch_batch_to_tiled(const void* src, int graphs, int n, int l, int k, void* dst, bool real,
                                  cudaStream_t stream) {
    if (real)
        batch_to_tiled_kernel<true><<<dim3(4, graphs), 256, 0, stream>>>((const double2*)src, n, l, k, dst);
    else
        batch_to_tiled_kernel<false><<<dim3(4, graphs), 256, 0, stream>>>((const double2*)src, n, l, k, dst);
    return cudaGetLastError();
}

#define FGB_BATCH_HEADS(MACRO) \
    switch (heads) {           \
        case 1: MACRO(1); break; \
        case 2: MACRO(2); break; \
        case 3: MACRO(3); break; \
        default: MACRO(4); break; \
    }

cudaError_t launch_batch_forward(const void* slabs, int graphs, int n, int l, const double* coef, int heads,
                                 const void* x, int ch, void* y, bool real, cudaStream_t stream) {
    // 2: the Y phase on the tensor cores (default); 0: the FFMA form. Measured at config 5: both
    // 0.64 ms -- the per-graph power stream, not the Y phase, bounds the kernel; a two-CTA-per-SM
    // FFMA form (0.65 ms) and a persistent warp-specialised form streaming across graphs (0.78 ms)
    // were tried and dropped.
    static const int fwd_form = [] {
        const char* e = std::getenv("FGFRFT_BATCH_FWD");
        return e ? std::atoi(e) : 3;
    }();
    // 3 (default): the persistent tcgen05 kernel for the config-5 shape (real F, n = 64, 64 channels)
    if (real && fwd_form == 3 && tc_shape_ok(n, ch, x, y)) {
        int stages = 0;
        const size_t sm = batch_tc_fwd_smem(l, heads, &stages);
        if (stages < 3) return cudaErrorInvalidValue;
        const int grid = graphs < FGFRFT_SMS ? graphs : FGFRFT_SMS;
#define FGB_BFT(HV)                                                                                            \
    {                                                                                                          \
        static PerDeviceOnce attr;                                                                             \
        cudaError_t e = attr.run([] {                                                                          \
            return cudaFuncSetAttribute(batch_fwd_tc_kernel<HV>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                        227 * 1024);                                                           \
        });                                                                                                    \
        if (e != cudaSuccess) return e;                                                                        \
        batch_fwd_tc_kernel<HV><<<grid, kTcThreads, sm, stream>>>((const float*)slabs, l,                      \
                                                                  batch_coef_f(coef, graphs * HV, l),          \
                                                                  (const float2*)x, (float2*)y, graphs, stages); \
    }
        FGB_BATCH_HEADS(FGB_BFT)
#undef FGB_BFT
        return cudaGetLastError();
    }
    if (real && fwd_form == 2) {
        const size_t sm = batch_forward_mma_smem_bytes(l, heads);
#define FGB_BFM(HV)                                                                                            \
    {                                                                                                          \
        static PerDeviceOnce attr;                                                                             \
        cudaError_t e = attr.run([] {                                                                          \
            return cudaFuncSetAttribute(batch_forward_mma_kernel<HV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                        227 * 1024);                                                           \
        });                                                                                                    \
        if (e != cudaSuccess) return e;                                                                        \
        batch_forward_mma_kernel<HV><<<graphs, kBTh, sm, stream>>>((const float*)slabs, n, l, coef,             \
                                                                   (const float2*)x, ch, (float2*)y);          \
    }
        if (sm > 227 * 1024) return cudaErrorInvalidValue;
        FGB_BATCH_HEADS(FGB_BFM)
#undef FGB_BFM
        return cudaGetLastError();
    }
    const size_t smem = batch_smem_bytes(l);
#define FGB_BF(HV)                                                                                             \
    {                                                                                                          \
        auto kern = real ? batch_forward_kernel<HV, true> : batch_forward_kernel<HV, false>;                    \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
        if (e != cudaSuccess) return e;                                                                        \
        kern<<<graphs, kBTh, smem, stream>>>(slabs, n, l, coef, (const float2*)x, ch, (float2*)y);              \
    }
    FGB_BATCH_HEADS(FGB_BF)
#undef FGB_BF
    return cudaGetLastError();
}

cudaError_t launch_batch_dlda(const void* slabs, int graphs, int n, int l, const double* coef, int heads,
                              const void* gcot, const void* x, int ch, double* dlda, bool real, cudaStream_t stream) {
    static const int form = [] {
        const char* e = std::getenv("FGFRFT_BATCH_DLDA");
        return e ? std::atoi(e) : 3;
    }();
    if (real && form == 3 && tc_shape_ok(n, ch, x, gcot)) {
        int stages = 0;
        const size_t sm = batch_tc_dlda_smem(l, heads, &stages);
        if (stages < 3) return cudaErrorInvalidValue;
        const int grid = graphs < FGFRFT_SMS ? graphs : FGFRFT_SMS;
#define FGB_BDT(HV)                                                                                            \
    {                                                                                                          \
        static PerDeviceOnce attr;                                                                             \
        cudaError_t e = attr.run([] {                                                                          \
            return cudaFuncSetAttribute(batch_dlda_tc_kernel<HV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                        227 * 1024);                                                           \
        });                                                                                                    \
        if (e != cudaSuccess) return e;                                                                        \
        batch_dlda_tc_kernel<HV><<<grid, kTcThreads, sm, stream>>>((const float*)slabs, l,                     \
                                                                   batch_coef_f(coef, graphs * HV, l),         \
                                                                   (const float2*)gcot, (const float2*)x,      \
                                                                   dlda, graphs, stages);                      \
    }
        FGB_BATCH_HEADS(FGB_BDT)
#undef FGB_BDT
        return cudaGetLastError();
    }
    const size_t smem = batch_smem_bytes(l);
#define FGB_BD(HV)                                                                                            \
    {                                                                                                         \
        auto kern = real ? batch_dlda_kernel<HV, true> : batch_dlda_kernel<HV, false>;                        \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
        if (e != cudaSuccess) return e;                                                                       \
        kern<<<graphs, kBTh, smem, stream>>>(slabs, n, l, coef, (const float2*)gcot, (const float2*)x, ch,    \
                                             dlda);                                                           \
    }
    FGB_BATCH_HEADS(FGB_BD)
#undef FGB_BD
    return cudaGetLastError();
}

int batch_max_heads() { return kBMaxHeads; }
int batch_max_channels() { return kBMaxCh; }
int batch_max_n() { return kBN; }

}  // namespace fgb
