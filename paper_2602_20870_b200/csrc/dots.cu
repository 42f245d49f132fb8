// dots.cu -- K4: per-power reductions for the order gradient.
//
//   s_k = Re<M, F^k>,  s_{-k} = Re<M, (F^k)^H>,  s_0 = Re tr M,   k = 1..L,
//
// so that with M = G X^H, Re<G, F^k X> = s_k and dL/dalpha = sum_k c'_k(alpha) s_k -- the
// quantity the reference forms as 2/N^2 Re sum conj(b) o (dQ X) (learn.hpp:88-92) and as the
// two Re<.,.> terms of the fast denoise engine (learn.hpp:328-337). One CTA owns a 32x32 tile
// pair {(I,J),(J,I)} of every power and of M (the same TMA ring as synth.cu), so each cache
// byte crosses HBM once; per power the CTA reduces with warp shuffles and writes one partial
// per (order, k). A second kernel sums the partials over tile pairs in a fixed order, so the
// result is deterministic (bit-identical across runs; SPEC determinism contract).
#include "common.cuh"

namespace fgb {

constexpr int kDotStages = 4, kDotThreads = 256;

size_t dots_smem_bytes(int l, int ac, int elem_bytes) {
    return (size_t)kDotStages * 2 * kTileElems * elem_bytes + kDotStages * 8 + (size_t)l * 8 * ac * 2 * sizeof(double) +
           16;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// slabs: tiled layout (common.cuh). partial layout: [a][2l+1][pair] (pairs contiguous so the
// fixed-order reduction over pairs is coalesced).
__device__ __forceinline__ double2 to_d2(const double2& v) { return v; }
__device__ __forceinline__ double2 to_d2(const float2& v) { return make_double2((double)v.x, (double)v.y); }

template <typename R, int AC>
__global__ void __launch_bounds__(kDotThreads, 1)
power_dots_kernel(const cplx_t<R>* __restrict__ slabs, int n, int l, int64_t slab_elems,
                  const cplx_t<R>* __restrict__ m, int64_t m_stride, int n_alpha, int n_achunks,
                  double* __restrict__ partial, int nt, int npairs) {
    using C = cplx_t<R>;
    constexpr int T = kTile, S = kDotStages;
    extern __shared__ __align__(128) unsigned char smem[];
    C* tiles = reinterpret_cast<C*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * 2 * kTileElems * sizeof(C));
    double* red = reinterpret_cast<double*>(full + S);  // [k-1][warp][a][2]

    const int chunk = blockIdx.x % n_achunks;
    const int pair = blockIdx.x / n_achunks;
    int I, J;
    pair_of(pair, I, J);
    const int a0 = chunk * AC;
    const int na = min(AC, n_alpha - a0);
    const int bi = min(T, n - I * T), bj = min(T, n - J * T);
    const bool diag = (I == J);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = lane;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t tile_bytes = (uint32_t)(kTileElems * sizeof(C));
    const bool stream_once = n_achunks == 1;
    const uint64_t pol = policy_evict_first();
    const int64_t off1 = tile_base(I, J, nt), off2 = tile_base(J, I, nt);
    auto issue = [&](int k, int s) {  // one thread: one bulk copy per 32x32 tile
        mbar_arrive_expect_tx(&full[s], (diag ? 1 : 2) * tile_bytes);
        const C* slab = slabs + (int64_t)(k - 1) * slab_elems;
        C* t1 = tiles + (size_t)(s * 2) * kTileElems;
        if (stream_once) {
            bulk_g2s_hint(t1, slab + off1, tile_bytes, &full[s], pol);
            if (!diag) bulk_g2s_hint(t1 + kTileElems, slab + off2, tile_bytes, &full[s], pol);
        } else {
            bulk_g2s(t1, slab + off1, tile_bytes, &full[s]);
            if (!diag) bulk_g2s(t1 + kTileElems, slab + off2, tile_bytes, &full[s]);
        }
    };
    if (tid == 0)
        for (int s = 0; s < S && s < l; ++s) issue(s + 1, s);

    // M tiles for this pair, zero outside the matrix so garbage smem never contributes.
    double2 m1[4][AC], m2[4][AC];
    double s0[AC];
#pragma unroll
    for (int a = 0; a < AC; ++a) s0[a] = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int c = warp + 8 * i;
        const bool v = r < bi && c < bj;
#pragma unroll
        for (int a = 0; a < AC; ++a) {
            const C* ma = m + (int64_t)(a0 + (a < na ? a : 0)) * m_stride;
            const bool va = v && a < na;
            m1[i][a] = va ? to_d2(ma[(int64_t)(J * T + c) * n + I * T + r]) : make_double2(0.0, 0.0);
            m2[i][a] = (va && !diag) ? to_d2(ma[(int64_t)(I * T + r) * n + J * T + c]) : make_double2(0.0, 0.0);
            if (diag && r == c) s0[a] += m1[i][a].x;
        }
    }

    // Powers are processed in groups of G so that one group yields NV = 16 per-lane partial
    // sums (G powers x AC orders x {+,-}); a transposing warp reduction (15 + 1 shuffles for
    // 16 values instead of 5 per value) leaves lane v (and v+16) holding the warp total of
    // value v, which is written to the per-warp table `red`.
    constexpr int NV = 16, G = NV / (2 * AC);
    for (int k0 = 1; k0 <= l; k0 += G) {
        double v[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) v[q] = 0.0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int k = k0 + g;
            if (k > l) break;
            const int s = (k - 1) % S;
            mbar_wait(&full[s], ((k - 1) / S) & 1);
            const C* t1 = tiles + (size_t)(s * 2) * kTileElems;
            const C* t2 = diag ? t1 : t1 + kTileElems;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int c = warp + 8 * i;
                const double2 p1 = to_d2(t1[swz(r, c)]);  // P[I*T + r, J*T + c]
                const double2 p2 = to_d2(t2[swz(c, r)]);  // P[J*T + c, I*T + r]
#pragma unroll
                for (int a = 0; a < AC; ++a) {
                    double& sp = v[(g * AC + a) * 2 + 0];
                    double& sm = v[(g * AC + a) * 2 + 1];
                    // Re(conj(m) p) and Re(conj(m) conj(p^T))
                    sp = fma(m1[i][a].x, p1.x, fma(m1[i][a].y, p1.y, sp));
                    sm = fma(m1[i][a].x, p2.x, fma(-m1[i][a].y, p2.y, sm));
                    if (!diag) {
                        sp = fma(m2[i][a].x, p2.x, fma(m2[i][a].y, p2.y, sp));
                        sm = fma(m2[i][a].x, p1.x, fma(-m2[i][a].y, p1.y, sm));
                    }
                }
            }
            __syncthreads();
            if (tid == 0 && k + S <= l) issue(k + S, s);
        }
        // transposing reduction over offsets 8, 4, 2, 1: lane keeps the half selected by its bit
#pragma unroll
        for (int o = 8, half = NV / 2; o >= 1; o >>= 1, half >>= 1) {
            const bool hi = (lane & o) != 0;
#pragma unroll
            for (int q = 0; q < half; ++q) {
                const double send = hi ? v[q] : v[q + half];
                const double keep = hi ? v[q + half] : v[q];
                v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 16);
        const int q = lane & (NV - 1);  // value index now held by this lane
        const int g = q / (2 * AC), a = (q / 2) % AC, sgn = q & 1;
        if (lane < NV && k0 + g <= l) red[(((size_t)(k0 + g - 1) * 8 + warp) * AC + a) * 2 + sgn] = v[0];
    }
    __syncthreads();

    // s0 partial: warp reduce then fixed-order sum over warps through the (now idle) stage ring.
    double* s0buf = reinterpret_cast<double*>(tiles);
#pragma unroll
    for (int a = 0; a < AC; ++a) {
        const double v = warp_sum(s0[a]);
        if (lane == 0) s0buf[warp * AC + a] = v;
    }
    __syncthreads();
    const int width = 2 * l + 1;
    for (int idx = tid; idx < na * width; idx += kDotThreads) {
        const int a = idx / width, kk = idx % width;  // kk = k + l
        double acc = 0.0;
        if (kk == l) {
            for (int w = 0; w < 8; ++w) acc += s0buf[w * AC + a];
        } else {
            const int k = kk > l ? kk - l : l - kk;
            const int sel = kk > l ? 0 : 1;
            for (int w = 0; w < 8; ++w) acc += red[(((size_t)(k - 1) * 8 + w) * AC + a) * 2 + sel];
        }
        partial[((int64_t)(a0 + a) * width + kk) * npairs + pair] = acc;
    }
}

// out[a][kk] = sum over tile pairs of partial[a][kk][pair]: one block per (a, kk), a fixed
// strided split over 128 threads and a fixed shuffle tree -> deterministic.
__global__ void __launch_bounds__(128) reduce_pairs_kernel(const double* __restrict__ partial, int npairs,
                                                           double* __restrict__ out) {
    const double* row = partial + (int64_t)blockIdx.x * npairs;
    double acc = 0.0;
    for (int p = threadIdx.x; p < npairs; p += 128) acc += row[p];
    acc = warp_sum(acc);
    __shared__ double ws[4];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = (ws[0] + ws[1]) + (ws[2] + ws[3]);
}

size_t dots_partial_elems(int n, int l, int n_alpha) {
    const int nt = (int)ceil_div(n, kTile);
    return (size_t)(nt * (nt + 1) / 2) * n_alpha * (2 * l + 1);
}

// s_out (device): [n_alpha][2l+1]; partial: device scratch of dots_partial_elems().
// elem_bytes: 16 (complex128 cache and M) or 8 (complex64).
cudaError_t launch_power_dots(const void* slabs, int n, int l, const void* m, int64_t m_stride, int n_alpha,
                              double* partial, double* s_out, cudaStream_t stream, int elem_bytes) {
    const int nt = (int)ceil_div(n, kTile);
    const int npairs = nt * (nt + 1) / 2;
    const int ac = n_alpha >= 4 ? 4 : (n_alpha >= 2 ? 2 : 1);
    const int nchunks = (int)ceil_div(n_alpha, ac);
    const size_t smem = dots_smem_bytes(l, ac, elem_bytes);
    const int64_t slab = (int64_t)nt * nt * kTileElems;
    const dim3 grid((unsigned)((int64_t)nchunks * npairs));
#define FGB_DOTS_CASE(RT, ACV)                                                                               \
    {                                                                                                        \
        auto kern = power_dots_kernel<RT, ACV>;                                                              \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e != cudaSuccess) return e;                                                                      \
        kern<<<grid, kDotThreads, smem, stream>>>((const cplx_t<RT>*)slabs, n, l, slab, (const cplx_t<RT>*)m, \
                                                  m_stride, n_alpha, nchunks, partial, nt, npairs);          \
    }
    if (elem_bytes == 16) {
        if (ac == 4) FGB_DOTS_CASE(double, 4) else if (ac == 2) FGB_DOTS_CASE(double, 2) else FGB_DOTS_CASE(double, 1)
    } else {
        if (ac == 4) FGB_DOTS_CASE(float, 4) else if (ac == 2) FGB_DOTS_CASE(float, 2) else FGB_DOTS_CASE(float, 1)
    }
#undef FGB_DOTS_CASE
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int total = n_alpha * (2 * l + 1);
    reduce_pairs_kernel<<<(unsigned)total, 128, 0, stream>>>(partial, npairs, s_out);
    return cudaGetLastError();
}

// =====================================================================================
// Sweep variant on the FP64 tensor cores.
//
// For many orders the contraction is a GEMM with a huge K:
//   D[a][kk] = sum_e A[a][e] B[e][kk],  e = (position of the tile pair, re/im),
//   kk = (k, +): B = P_k(e)            -> s_{+k} = Re<M_a, P_k>
//   kk = (k, -): B = conj(P_k^T)(e)    -> s_{-k} = Re<M_a, P_k^H>
// One CTA owns a 32x32 tile pair for up to 64 orders x 64 powers and walks it in 4x4
// sub-square pairs (16 positions of tile (I,J) + their 16 transposed partners in (J,I)), so the
// transposed operand is always staged in the same block. Every byte of M and of the cache is
// read once per launch (no order chunking through L2). 8 warps = 2 (orders) x 4 (power terms),
// warp tile 32 x 32 of D, four m8n8k4 DMMAs per fragment pair and K4 step. Staging is 16-byte
// cp.async per element (one element = one position), 3-stage ring.
// =====================================================================================

constexpr int kDmA = 64;        // orders per launch (rows of D)
constexpr int kDmK = 64;        // powers per launch (kk = 128 columns of D)
constexpr int kDmLd = 34;       // complex elements per staged M row (32 + pad)
constexpr int kDmLdP = 36;      // power rows: [t=0: 16][pad 2][t=1: 16][pad 2] complex; 64-bit fragment
constexpr int kDmPT1 = 18;      // loads of one half-warp then hit 16 distinct bank pairs
constexpr int kDmStages = 3;
constexpr int kDmStage = kDmA * kDmLd + kDmK * kDmLdP;  // complex elements per stage

size_t dots_mma_smem_bytes() { return (size_t)kDmStages * kDmStage * 16; }

// partial layout: [pair][a (kDmA)][kk (2*kDmK)]
__global__ void __launch_bounds__(256, 1)
power_dots_mma_kernel(const double2* __restrict__ slabs, int n, int k_begin, int k_count, int64_t slab_elems,
                      const double2* __restrict__ m, int64_t m_stride, int n_alpha, double* __restrict__ partial,
                      int nt) {
    extern __shared__ __align__(128) unsigned char smem[];
    double2* stage_base = reinterpret_cast<double2*>(smem);
    const int pair = blockIdx.x;
    int I, J;
    pair_of(pair, I, J);
    const bool diag = (I == J);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wa = warp & 1, wk = warp >> 1;
    const int64_t b1 = tile_base(I, J, nt), b2 = tile_base(J, I, nt);

    // Stage block `blk` (sub-square r0 = 4*(blk%8), c0 = 4*(blk/8)) into ring slot `s`.
    // Row a (< kDmA) holds M_a at the 32 positions, row kDmA + k' holds P_{k_begin+k'}.
    // Position index p = t*16 + jj*4 + ii: t = 0 -> (I*32+r0+ii, J*32+c0+jj); t = 1 -> its
    // transpose (J*32+c0+jj, I*32+r0+ii).
    auto stage = [&](int blk, int s) {
        double2* st = stage_base + (size_t)s * kDmStage;
        const int r0 = 4 * (blk & 7), c0 = 4 * (blk >> 3);
        for (int idx = tid; idx < (kDmA + kDmK) * 32; idx += 256) {
            const int row = idx >> 5, p = idx & 31;
            const int t = p >> 4, jj = (p >> 2) & 3, ii = p & 3;
            const int li = r0 + ii, lj = c0 + jj;  // local (row, col) in tile (I,J)
            double2* dst = row < kDmA ? st + row * kDmLd + p
                                      : st + kDmA * kDmLd + (row - kDmA) * kDmLdP + t * kDmPT1 + (p & 15);
            if (row < kDmA) {
                const int a = row;
                const int gi = t == 0 ? I * 32 + li : J * 32 + lj;
                const int gj = t == 0 ? J * 32 + lj : I * 32 + li;
                const bool v = a < n_alpha && gi < n && gj < n && !(diag && t == 1);
                const double2* src = v ? m + (int64_t)a * m_stride + (int64_t)gj * n + gi : m;
                cp_async16(dst, src, v);
            } else {
                const int kq = row - kDmA;
                const bool v = kq < k_count;
                const double2* slab = slabs + (int64_t)(k_begin + (v ? kq : 0) - 1) * slab_elems;
                const double2* src = t == 0 ? slab + b1 + swz(li, lj) : slab + b2 + swz(lj, li);
                cp_async16(dst, src, v);
            }
        }
    };

    double d[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) d[i][j][0] = d[i][j][1] = 0.0;

    const int nblk = 64;
#pragma unroll
    for (int s = 0; s < kDmStages - 1; ++s) {
        stage(s, s);
        cp_async_commit();
    }
    for (int blk = 0; blk < nblk; ++blk) {
        cp_async_wait<kDmStages - 2>();
        __syncthreads();
        if (blk + kDmStages - 1 < nblk) stage(blk + kDmStages - 1, (blk + kDmStages - 1) % kDmStages);
        cp_async_commit();
        const double2* st = stage_base + (size_t)(blk % kDmStages) * kDmStage;
        const double* ms = reinterpret_cast<const double*>(st);
        const double* ps = reinterpret_cast<const double*>(st + kDmA * kDmLd);
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
            const int e = 4 * ks + t4;             // K index: (position p = e >> 1, component e & 1)
            const int p = e >> 1, comp = e & 1;
            const int tp = p >> 4, pl = p & 15;    // transposed partner: same pl, other half
            double a[4], b[4];
#pragma unroll
            for (int mb = 0; mb < 4; ++mb) a[mb] = ms[((32 * wa + 8 * mb + g) * kDmLd + p) * 2 + comp];
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) {
                const int kk = 32 * wk + 8 * nb + g;
                const int kq = kk >> 1;
                const double v = ps[(kq * kDmLdP + (tp ^ (kk & 1)) * kDmPT1 + pl) * 2 + comp];
                b[nb] = ((kk & 1) && comp) ? -v : v;
            }
#pragma unroll
            for (int mb = 0; mb < 4; ++mb)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) dmma884(d[mb][nb][0], d[mb][nb][1], a[mb], b[nb]);
        }
    }
    cp_async_wait<0>();
    double* out = partial + (int64_t)pair * kDmA * (2 * kDmK);
#pragma unroll
    for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
            const int a = 32 * wa + 8 * mb + g;
            const int kk = 32 * wk + 8 * nb + 2 * t4;
            *reinterpret_cast<double2*>(out + a * (2 * kDmK) + kk) = make_double2(d[mb][nb][0], d[mb][nb][1]);
        }
}

// s_out[a][k + l] for k = +-(k_begin .. k_begin+k_count-1): fixed-order sum over pairs.
__global__ void __launch_bounds__(128) reduce_mma_pairs_kernel(const double* __restrict__ partial, int npairs,
                                                               int n_alpha, int k_begin, int k_count, int l,
                                                               double* __restrict__ s_out) {
    const int a = blockIdx.x / (2 * k_count), kk = blockIdx.x % (2 * k_count);
    double acc = 0.0;
    for (int p = threadIdx.x; p < npairs; p += 128) acc += partial[((int64_t)p * kDmA + a) * (2 * kDmK) + kk];
    acc = warp_sum(acc);
    __shared__ double ws[4];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        const int k = k_begin + (kk >> 1);
        const int col = (kk & 1) ? l - k : l + k;
        s_out[(int64_t)a * (2 * l + 1) + col] = (ws[0] + ws[1]) + (ws[2] + ws[3]);
    }
}

// s_out[a][l] = Re tr(M_a), fixed order.
__global__ void __launch_bounds__(128) trace_re_kernel(const double2* __restrict__ m, int64_t m_stride, int n, int l,
                                                       double* __restrict__ s_out) {
    const int a = blockIdx.x;
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += 128) acc += m[(int64_t)a * m_stride + (int64_t)i * n + i].x;
    acc = warp_sum(acc);
    __shared__ double ws[4];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) s_out[(int64_t)a * (2 * l + 1) + l] = (ws[0] + ws[1]) + (ws[2] + ws[3]);
}

size_t dots_mma_partial_elems(int n) {
    const int nt = (int)ceil_div(n, kTile);
    return (size_t)(nt * (nt + 1) / 2) * kDmA * 2 * kDmK;
}

int dots_mma_max_orders() { return kDmA; }

// n_alpha <= 64. s_out (device): [n_alpha][2l+1]. Launches: ceil(l/64) x (dots + reduce) + trace.
cudaError_t launch_power_dots_mma(const void* slabs, int n, int l, const void* m, int64_t m_stride, int n_alpha,
                                  double* partial, double* s_out, cudaStream_t stream, int* launches) {
    const int nt = (int)ceil_div(n, kTile);
    const int npairs = nt * (nt + 1) / 2;
    const int64_t slab = (int64_t)nt * nt * kTileElems;
    const size_t smem = dots_mma_smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(power_dots_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int nl = 0;
    for (int k0 = 1; k0 <= l; k0 += kDmK) {
        const int kc = min(kDmK, l - k0 + 1);
        power_dots_mma_kernel<<<npairs, 256, smem, stream>>>((const double2*)slabs, n, k0, kc, slab,
                                                             (const double2*)m, m_stride, n_alpha, partial, nt);
        reduce_mma_pairs_kernel<<<n_alpha * 2 * kc, 128, 0, stream>>>(partial, npairs, n_alpha, k0, kc, l, s_out);
        nl += 2;
    }
    trace_re_kernel<<<n_alpha, 128, 0, stream>>>((const double2*)m, m_stride, n, l, s_out);
    if (launches) *launches = nl + 1;
    return cudaGetLastError();
}

}  // namespace fgb
