// shard.cu -- row-slab sharding of the power cache for multi-GPU runs.
//
// Rank g owns rows R = [r0, r1) of the output. It stores, for every power k, the row panel
// P_k[R, :] and the column panel P_k[:, R] (tiled + swizzled as in common.cuh), i.e. the rows of
// both F^k and F^{-k} = (F^k)^H -- the north star's 2L+1-slab layout split by rows. With F
// replicated, every quantity a rank needs is local:
//   Q[R, :]      = c_0 I[R,:] + sum_k a_k P_k[R,:] + b_k conj(P_k[:,R])^T      (synth_rows_kernel)
//   Y[R, :]      = Q[R, :] X                                                  (DMMA GEMM)
//   s_k partial  = Re<M[R,:], P_k[R,:]>,  s_{-k} = Re<M[R,:], conj(P_k[:,R])^T>, M[R,:] = G[R,:] X^H
// so the only collectives are an all-reduce of the 2L+1 partials (and the loss) and a gather
// of Y's rows. Panel build: P_k[R,:] = P_{k-1}[R,:] F and P_k[:,R] = F P_{k-1}[:,R] (powers of F
// commute), both on the DMMA GEMM.
//
// Tiled panel layouts: row panel tile (i, J) (i = local block row) at ((J * nI) + i) * 1024;
// column panel tile (J, i) at ((i * nt) + J) * 1024.
#include "common.cuh"

namespace fgb {

constexpr int kRowStages = 4;

// Rectangular column-major (m x ncols, ld) -> tiled with tile (I, J) at (J * ntm + I) * 1024.
template <typename T>
__global__ void __launch_bounds__(256) rect_to_tiled_kernel(const T* __restrict__ src, int64_t ld, int m, int ncols,
                                                            T* __restrict__ dst, int ntm) {
    const int I = blockIdx.x % ntm, J = blockIdx.x / ntm;
    const int r = threadIdx.x & 31, w = threadIdx.x >> 5;
    T* t = dst + ((int64_t)J * ntm + I) * kTileElems;
    const int row = I * kTile + r;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int c = w + 8 * i, col = J * kTile + c;
        t[swz(r, c)] = (row < m && col < ncols) ? src[(int64_t)col * ld + row] : T{};
    }
}

cudaError_t launch_rect_to_tiled(const void* src, int64_t ld, int m, int ncols, void* dst, cudaStream_t stream,
                                 bool real) {
    const int ntm = (int)ceil_div(m, kTile), ntn = (int)ceil_div(ncols, kTile);
    if (real)
        rect_to_tiled_kernel<double><<<ntm * ntn, 256, 0, stream>>>((const double*)src, ld, m, ncols, (double*)dst,
                                                                    ntm);
    else
        rect_to_tiled_kernel<double2><<<ntm * ntn, 256, 0, stream>>>((const double2*)src, ld, m, ncols,
                                                                     (double2*)dst, ntm);
    return cudaGetLastError();
}

// q += a*p + b*conj(pt) without contraction (the reference's evaluation order).
__device__ __forceinline__ void pair_update_d(double2& q, double a, double b, const double2& p, const double2& pt) {
    q.x = __dadd_rn(q.x, __dadd_rn(__dmul_rn(a, p.x), __dmul_rn(b, pt.x)));
    q.y = __dadd_rn(q.y, __dadd_rn(__dmul_rn(a, p.y), __dmul_rn(b, -pt.y)));
}

__device__ __forceinline__ void pair_update_d(double& q, double a, double b, const double& p, const double& pt) {
    q = __dadd_rn(q, __dadd_rn(__dmul_rn(a, p), __dmul_rn(b, pt)));
}

__host__ __device__ inline size_t rows_smem_bytes(int l, int ac, int esz) {
    return (size_t)kRowStages * 2 * kTileElems * esz + kRowStages * 8 + (size_t)l * ac * 16 + (size_t)ac * 8 + 16;
}

template <typename T> __device__ __forceinline__ T zero_of(double v);
template <> __device__ __forceinline__ double2 zero_of<double2>(double v) { return make_double2(v, 0.0); }
template <> __device__ __forceinline__ double zero_of<double>(double v) { return v; }

// CTA per (order chunk, tile (I0 + i, J)); output rows panel (ld = rows).
template <typename T, int AC, bool OUTC>
__global__ void __launch_bounds__(256, 1)
synth_rows_kernel(const T* __restrict__ rowp, const T* __restrict__ colp, int64_t panel_elems, int n,
                  int r0, int rows, int l_used, const double* __restrict__ coef, int coef_ld, int n_alpha,
                  int n_achunks, void* __restrict__ out, int64_t out_stride, int nI, int nt) {
    constexpr int S = kRowStages;
    extern __shared__ __align__(128) unsigned char smem[];
    T* tiles = reinterpret_cast<T*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * 2 * kTileElems * sizeof(T));
    double2* cs = reinterpret_cast<double2*>(full + S);
    double* c0s = reinterpret_cast<double*>(cs + (size_t)l_used * AC);
    const int chunk = blockIdx.x % n_achunks, tidx = blockIdx.x / n_achunks;
    const int i = tidx % nI, J = tidx / nI;
    const int a0 = chunk * AC, na = min(AC, n_alpha - a0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lc = l_used;
    for (int idx = tid; idx < l_used * AC; idx += 256) {
        const int k = idx / AC + 1, a = idx % AC;
        double ak = 0.0, bk = 0.0;
        if (a < na) {
            ak = coef[(size_t)(a0 + a) * coef_ld + lc + k];
            bk = coef[(size_t)(a0 + a) * coef_ld + lc - k];
        }
        cs[idx] = make_double2(ak, bk);
    }
    if (tid < AC) c0s[tid] = tid < na ? coef[(size_t)(a0 + tid) * coef_ld + lc] : 0.0;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint32_t tb = kTileElems * sizeof(T);
    const uint64_t pol = policy_evict_first();
    const int64_t off1 = ((int64_t)J * nI + i) * kTileElems, off2 = ((int64_t)i * nt + J) * kTileElems;
    auto issue = [&](int k, int s) {
        mbar_arrive_expect_tx(&full[s], 2 * tb);
        T* t1 = tiles + (size_t)(s * 2) * kTileElems;
        bulk_g2s_hint(t1, rowp + (int64_t)(k - 1) * panel_elems + off1, tb, &full[s], pol);
        bulk_g2s_hint(t1 + kTileElems, colp + (int64_t)(k - 1) * panel_elems + off2, tb, &full[s], pol);
    };
    if (tid == 0)
        for (int s = 0; s < S && s < l_used; ++s) issue(s + 1, s);
    const int gI = r0 / kTile + i;  // global block row
    const int r = lane;
    T q[4][AC];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int c = warp + 8 * u;
#pragma unroll
        for (int a = 0; a < AC; ++a) q[u][a] = zero_of<T>((gI == J && r == c) ? c0s[a] : 0.0);
    }
    for (int k = 1; k <= l_used; ++k) {
        const int s = (k - 1) % S;
        mbar_wait(&full[s], ((k - 1) / S) & 1);
        const T* t1 = tiles + (size_t)(s * 2) * kTileElems;
        const T* t2 = t1 + kTileElems;
        double2 ab[AC];
#pragma unroll
        for (int a = 0; a < AC; ++a) ab[a] = cs[(k - 1) * AC + a];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = warp + 8 * u;
            const T p1 = t1[swz(r, c)];  // P[gI*32 + r, J*32 + c]
            const T p2 = t2[swz(c, r)];  // P[J*32 + c, gI*32 + r]
#pragma unroll
            for (int a = 0; a < AC; ++a) pair_update_d(q[u][a], ab[a].x, ab[a].y, p1, p2);
        }
        __syncthreads();
        if (tid == 0 && k + S <= l_used) issue(k + S, s);
    }
    const int lrow = i * kTile + r;
#pragma unroll
    for (int a = 0; a < AC; ++a) {
        if (a >= na) break;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int col = J * kTile + warp + 8 * u;
            if (lrow < rows && col < n) {
                const int64_t o = (int64_t)(a0 + a) * out_stride + (int64_t)col * rows + lrow;
                if constexpr (OUTC && sizeof(T) == 8) reinterpret_cast<double2*>(out)[o] = make_double2(q[u][a], 0.0);
                else reinterpret_cast<T*>(out)[o] = q[u][a];
            }
        }
    }
}

// real: real panels; out_complex: write complex128 (API output) even from real panels.
cudaError_t launch_synth_rows(const void* rowp, const void* colp, int n, int r0, int rows, int l_used,
                              const double* coef_dev, int n_alpha, void* out, cudaStream_t stream, bool real,
                              bool out_complex) {
    const int nI = (int)ceil_div(rows, kTile), nt = (int)ceil_div(n, kTile);
    const int64_t panel = (int64_t)nI * nt * kTileElems;
    const int ac = n_alpha >= 4 ? 4 : (n_alpha >= 2 ? 2 : 1);
    const int nch = (int)ceil_div(n_alpha, ac);
    const size_t smem = rows_smem_bytes(l_used, ac, real ? 8 : 16);
    const dim3 grid((unsigned)((int64_t)nch * nI * nt));
#define FGB_ROWS_CASE(TT, ACV, OC)                                                                           \
    {                                                                                                        \
        auto kern = synth_rows_kernel<TT, ACV, OC>;                                                          \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e != cudaSuccess) return e;                                                                      \
        kern<<<grid, 256, smem, stream>>>((const TT*)rowp, (const TT*)colp, panel, n, r0, rows, l_used,      \
                                          coef_dev, 2 * l_used + 1, n_alpha, nch, out, (int64_t)rows * n, nI, \
                                          nt);                                                               \
    }
    if (!real) {
        if (ac == 4) FGB_ROWS_CASE(double2, 4, true) else if (ac == 2) FGB_ROWS_CASE(double2, 2, true) else FGB_ROWS_CASE(double2, 1, true)
    } else if (out_complex) {
        if (ac == 4) FGB_ROWS_CASE(double, 4, true) else if (ac == 2) FGB_ROWS_CASE(double, 2, true) else FGB_ROWS_CASE(double, 1, true)
    } else {
        if (ac == 4) FGB_ROWS_CASE(double, 4, false) else if (ac == 2) FGB_ROWS_CASE(double, 2, false) else FGB_ROWS_CASE(double, 1, false)
    }
#undef FGB_ROWS_CASE
    return cudaGetLastError();
}

// Partial dots over the rank's rows: per tile (i, J): s_+ = Re<M, P>, s_- = Re<M, conj(P^T)>.
// partial layout [a][2l+1][tile]; M rows panel (ld = rows).
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double re_dot(const double2& m, const double2& p, double acc) {
    return fma(m.x, p.x, fma(m.y, p.y, acc));
}
__device__ __forceinline__ double re_dot_conj(const double2& m, const double2& p, double acc) {
    return fma(m.x, p.x, fma(-m.y, p.y, acc));
}
__device__ __forceinline__ double re_dot(const double& m, const double& p, double acc) { return fma(m, p, acc); }
__device__ __forceinline__ double re_dot_conj(const double& m, const double& p, double acc) { return fma(m, p, acc); }
__device__ __forceinline__ double re_of(const double2& v) { return v.x; }
__device__ __forceinline__ double re_of(const double& v) { return v; }

template <typename T, int AC>
__global__ void __launch_bounds__(256, 1)
dots_rows_kernel(const T* __restrict__ rowp, const T* __restrict__ colp, int64_t panel_elems, int n,
                 int r0, int rows, int l, const T* __restrict__ m, int64_t m_stride, int n_alpha,
                 int n_achunks, double* __restrict__ partial, int nI, int nt) {
    constexpr int S = kRowStages;
    extern __shared__ __align__(128) unsigned char smem[];
    T* tiles = reinterpret_cast<T*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * 2 * kTileElems * sizeof(T));
    double* red = reinterpret_cast<double*>(full + S);  // [k-1][warp][a][2]
    const int chunk = blockIdx.x % n_achunks, tidx = blockIdx.x / n_achunks;
    const int i = tidx % nI, J = tidx / nI;
    const int ntiles = nI * nt;
    const int a0 = chunk * AC, na = min(AC, n_alpha - a0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, r = lane;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint32_t tb = kTileElems * sizeof(T);
    const uint64_t pol = policy_evict_first();
    const int64_t off1 = ((int64_t)J * nI + i) * kTileElems, off2 = ((int64_t)i * nt + J) * kTileElems;
    auto issue = [&](int k, int s) {
        mbar_arrive_expect_tx(&full[s], 2 * tb);
        T* t1 = tiles + (size_t)(s * 2) * kTileElems;
        bulk_g2s_hint(t1, rowp + (int64_t)(k - 1) * panel_elems + off1, tb, &full[s], pol);
        bulk_g2s_hint(t1 + kTileElems, colp + (int64_t)(k - 1) * panel_elems + off2, tb, &full[s], pol);
    };
    if (tid == 0)
        for (int s = 0; s < S && s < l; ++s) issue(s + 1, s);
    const int gI = r0 / kTile + i;
    T mv[4][AC];
    double s0[AC];
#pragma unroll
    for (int a = 0; a < AC; ++a) s0[a] = 0.0;
    const int lrow = i * kTile + r;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int c = warp + 8 * u, col = J * kTile + c;
#pragma unroll
        for (int a = 0; a < AC; ++a) {
            const bool v = a < na && lrow < rows && col < n;
            mv[u][a] = v ? m[(int64_t)(a0 + a) * m_stride + (int64_t)col * rows + lrow] : T{};
            if (gI == J && r == c) s0[a] += re_of(mv[u][a]);
        }
    }
    for (int k = 1; k <= l; ++k) {
        const int s = (k - 1) % S;
        mbar_wait(&full[s], ((k - 1) / S) & 1);
        const T* t1 = tiles + (size_t)(s * 2) * kTileElems;
        const T* t2 = t1 + kTileElems;
        double sp[AC], sm[AC];
#pragma unroll
        for (int a = 0; a < AC; ++a) sp[a] = sm[a] = 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = warp + 8 * u;
            const T p1 = t1[swz(r, c)];
            const T p2 = t2[swz(c, r)];
#pragma unroll
            for (int a = 0; a < AC; ++a) {
                sp[a] = re_dot(mv[u][a], p1, sp[a]);
                sm[a] = re_dot_conj(mv[u][a], p2, sm[a]);
            }
        }
#pragma unroll
        for (int a = 0; a < AC; ++a) {
            const double vp = warp_sum_d(sp[a]), vm = warp_sum_d(sm[a]);
            if (lane == 0) {
                red[(((size_t)(k - 1) * 8 + warp) * AC + a) * 2 + 0] = vp;
                red[(((size_t)(k - 1) * 8 + warp) * AC + a) * 2 + 1] = vm;
            }
        }
        __syncthreads();
        if (tid == 0 && k + S <= l) issue(k + S, s);
    }
    double* s0buf = reinterpret_cast<double*>(tiles);
#pragma unroll
    for (int a = 0; a < AC; ++a) {
        const double v = warp_sum_d(s0[a]);
        if (lane == 0) s0buf[warp * AC + a] = v;
    }
    __syncthreads();
    const int width = 2 * l + 1;
    for (int idx = tid; idx < na * width; idx += 256) {
        const int a = idx / width, kk = idx % width;
        double acc = 0.0;
        if (kk == l) {
            for (int w = 0; w < 8; ++w) acc += s0buf[w * AC + a];
        } else {
            const int k = kk > l ? kk - l : l - kk, sel = kk > l ? 0 : 1;
            for (int w = 0; w < 8; ++w) acc += red[(((size_t)(k - 1) * 8 + w) * AC + a) * 2 + sel];
        }
        partial[((int64_t)(a0 + a) * width + kk) * ntiles + tidx] = acc;
    }
}

__global__ void __launch_bounds__(128) reduce_rows_kernel(const double* __restrict__ partial, int ntiles,
                                                          double* __restrict__ out) {
    const double* row = partial + (int64_t)blockIdx.x * ntiles;
    double acc = 0.0;
    for (int p = threadIdx.x; p < ntiles; p += 128) acc += row[p];
    acc = warp_sum_d(acc);
    __shared__ double ws[4];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = (ws[0] + ws[1]) + (ws[2] + ws[3]);
}

size_t dots_rows_partial_elems(int n, int rows, int l, int n_alpha) {
    return (size_t)ceil_div(rows, kTile) * ceil_div(n, kTile) * n_alpha * (2 * l + 1);
}

cudaError_t launch_dots_rows(const void* rowp, const void* colp, int n, int r0, int rows, int l, const void* m,
                             int64_t m_stride, int n_alpha, double* partial, double* s_out, cudaStream_t stream,
                             bool real) {
    const int nI = (int)ceil_div(rows, kTile), nt = (int)ceil_div(n, kTile);
    const int64_t panel = (int64_t)nI * nt * kTileElems;
    const int ac = n_alpha >= 4 ? 4 : (n_alpha >= 2 ? 2 : 1);
    const int nch = (int)ceil_div(n_alpha, ac);
    const size_t esz = real ? 8 : 16;
    const size_t smem = (size_t)kRowStages * 2 * kTileElems * esz + kRowStages * 8 + (size_t)l * 8 * ac * 2 * 8 + 16;
    const dim3 grid((unsigned)((int64_t)nch * nI * nt));
#define FGB_DR_CASE(TT, ACV)                                                                                 \
    {                                                                                                        \
        auto kern = dots_rows_kernel<TT, ACV>;                                                               \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e != cudaSuccess) return e;                                                                      \
        kern<<<grid, 256, smem, stream>>>((const TT*)rowp, (const TT*)colp, panel, n, r0, rows, l,           \
                                          (const TT*)m, m_stride, n_alpha, nch, partial, nI, nt);            \
    }
    if (real) {
        if (ac == 4) FGB_DR_CASE(double, 4) else if (ac == 2) FGB_DR_CASE(double, 2) else FGB_DR_CASE(double, 1)
    } else {
        if (ac == 4) FGB_DR_CASE(double2, 4) else if (ac == 2) FGB_DR_CASE(double2, 2) else FGB_DR_CASE(double2, 1)
    }
#undef FGB_DR_CASE
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    reduce_rows_kernel<<<n_alpha * (2 * l + 1), 128, 0, stream>>>(partial, nI * nt, s_out);
    return cudaGetLastError();
}

// Rows [r0, r0 + rows) of na blocks of n x b complex128 (column-major, block stride n b) from the
// local full buffer to every peer's buffer (NVLink P2P stores): the all-gather of a row-sharded
// result for the GEMMs that cannot write peers from their epilogue (DMMA path).
__global__ void rows_push_kernel(const double2* __restrict__ src, int64_t n, int r0, int rows, int64_t cols,
                                 double2* const* __restrict__ dst, int ndst) {
    const int64_t total = (int64_t)rows * cols;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = idx / rows, i = idx - j * rows;
        const int64_t o = j * n + r0 + i;
        const double2 v = src[o];
        for (int d = 0; d < ndst; ++d) dst[d][o] = v;
    }
}

cudaError_t launch_rows_push(const void* src, int64_t n, int r0, int rows, int64_t cols, void* const* dst_dev,
                             int ndst, cudaStream_t stream) {
    if (ndst <= 0 || rows <= 0 || cols <= 0) return cudaSuccess;
    rows_push_kernel<<<8 * FGFRFT_SMS, 256, 0, stream>>>((const double2*)src, n, r0, rows, cols,
                                                         (double2* const*)dst_dev, ndst);
    return cudaGetLastError();
}

}  // namespace fgb
