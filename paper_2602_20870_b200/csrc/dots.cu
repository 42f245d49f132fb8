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

size_t dots_smem_bytes(int l, int ac) {
    return (size_t)kDotStages * 2 * kTileElems * 16 + kDotStages * 8 + (size_t)l * 8 * ac * 2 * sizeof(double) + 16;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// slabs: tiled layout (common.cuh). partial layout: [a][2l+1][pair] (pairs contiguous so the
// fixed-order reduction over pairs is coalesced).
template <int AC>
__global__ void __launch_bounds__(kDotThreads, 1)
power_dots_kernel(const double2* __restrict__ slabs, int n, int l, int64_t slab_elems,
                  const double2* __restrict__ m, int64_t m_stride, int n_alpha, int n_achunks,
                  double* __restrict__ partial, int nt, int npairs) {
    constexpr int T = kTile, S = kDotStages;
    extern __shared__ __align__(128) unsigned char smem[];
    double2* tiles = reinterpret_cast<double2*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * 2 * kTileElems * 16);
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

    const uint32_t tile_bytes = (uint32_t)(kTileElems * 16);
    const bool stream_once = n_achunks == 1;
    const uint64_t pol = policy_evict_first();
    const int64_t off1 = tile_base(I, J, nt), off2 = tile_base(J, I, nt);
    auto issue = [&](int k, int s) {  // one thread: one bulk copy per 32x32 tile
        mbar_arrive_expect_tx(&full[s], (diag ? 1 : 2) * tile_bytes);
        const double2* slab = slabs + (int64_t)(k - 1) * slab_elems;
        double2* t1 = tiles + (size_t)(s * 2) * kTileElems;
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
            const double2* ma = m + (int64_t)(a0 + (a < na ? a : 0)) * m_stride;
            const bool va = v && a < na;
            m1[i][a] = va ? ma[(int64_t)(J * T + c) * n + I * T + r] : make_double2(0.0, 0.0);
            m2[i][a] = (va && !diag) ? ma[(int64_t)(I * T + r) * n + J * T + c] : make_double2(0.0, 0.0);
            if (diag && r == c) s0[a] += m1[i][a].x;
        }
    }

    for (int k = 1; k <= l; ++k) {
        const int s = (k - 1) % S;
        mbar_wait(&full[s], ((k - 1) / S) & 1);
        const double2* t1 = tiles + (size_t)(s * 2) * kTileElems;
        const double2* t2 = diag ? t1 : t1 + kTileElems;
        double sp[AC], sm[AC];
#pragma unroll
        for (int a = 0; a < AC; ++a) sp[a] = sm[a] = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = warp + 8 * i;
            const double2 p1 = t1[swz(r, c)];  // P[I*T + r, J*T + c]
            const double2 p2 = t2[swz(c, r)];  // P[J*T + c, I*T + r]
#pragma unroll
            for (int a = 0; a < AC; ++a) {
                // Re(conj(m) p) and Re(conj(m) conj(p^T))
                sp[a] = fma(m1[i][a].x, p1.x, fma(m1[i][a].y, p1.y, sp[a]));
                sm[a] = fma(m1[i][a].x, p2.x, fma(-m1[i][a].y, p2.y, sm[a]));
                if (!diag) {
                    sp[a] = fma(m2[i][a].x, p2.x, fma(m2[i][a].y, p2.y, sp[a]));
                    sm[a] = fma(m2[i][a].x, p1.x, fma(-m2[i][a].y, p1.y, sm[a]));
                }
            }
        }
#pragma unroll
        for (int a = 0; a < AC; ++a) {
            const double vp = warp_sum(sp[a]);
            const double vm = warp_sum(sm[a]);
            if (lane == 0) {
                red[(((size_t)(k - 1) * 8 + warp) * AC + a) * 2 + 0] = vp;
                red[(((size_t)(k - 1) * 8 + warp) * AC + a) * 2 + 1] = vm;
            }
        }
        __syncthreads();
        if (tid == 0 && k + S <= l) issue(k + S, s);
    }

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
cudaError_t launch_power_dots(const void* slabs, int n, int l, const void* m, int64_t m_stride, int n_alpha,
                              double* partial, double* s_out, cudaStream_t stream) {
    const int nt = (int)ceil_div(n, kTile);
    const int npairs = nt * (nt + 1) / 2;
    const int ac = n_alpha >= 4 ? 4 : (n_alpha >= 2 ? 2 : 1);
    const int nchunks = (int)ceil_div(n_alpha, ac);
    const size_t smem = dots_smem_bytes(l, ac);
    const int64_t slab = (int64_t)nt * nt * kTileElems;
    const dim3 grid((unsigned)((int64_t)nchunks * npairs));
#define FGB_DOTS_CASE(ACV)                                                                                   \
    {                                                                                                        \
        auto kern = power_dots_kernel<ACV>;                                                                  \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e != cudaSuccess) return e;                                                                      \
        kern<<<grid, kDotThreads, smem, stream>>>((const double2*)slabs, n, l, slab, (const double2*)m,     \
                                                  m_stride, n_alpha, nchunks, partial, nt, npairs);                  \
    }
    if (ac == 4) FGB_DOTS_CASE(4) else if (ac == 2) FGB_DOTS_CASE(2) else FGB_DOTS_CASE(1)
#undef FGB_DOTS_CASE
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int total = n_alpha * (2 * l + 1);
    reduce_pairs_kernel<<<(unsigned)total, 128, 0, stream>>>(partial, npairs, s_out);
    return cudaGetLastError();
}

}  // namespace fgb
