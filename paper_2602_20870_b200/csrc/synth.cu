// synth.cu -- K2: series synthesis Q = c_0 I + sum_{k=1..L'} (a_k F^k + b_k (F^k)^H).
//
// Replaces fgfrft_matrix / fgfrft_grad / detail::add_scaled_pair
// (proj/include/fgfrft/transform.hpp:21-34, 111-136). The reference walks 96x96 blocks and
// reads the transposed block of every power on the fly; here one CTA owns a 32x32 TILE PAIR
// {(I,J), (J,I)} and streams both tiles of every cached power through shared memory exactly
// once (TMA bulk copies, 4-stage mbarrier ring), producing Q[I,J] and Q[J,I] together. Every
// cache byte therefore crosses HBM once per launch: algorithmic bytes = (L' + A) n^2 s.
//
// Multi-order launches (A orders): a CTA accumulates AC orders in registers; CTAs of the
// ceil(A/AC) order chunks of one tile pair are adjacent in the grid, so the chunks after the
// first are served from L2. The cache is stored tiled + XOR-swizzled (common.cuh): each staged
// tile is ONE contiguous 16 KB bulk copy and both the direct and the transposed shared-memory
// reads are conflict free.
//
// Arithmetic: the reference's per-element update t = a*p_ij + b*conj(p_ji); q = q + t is
// evaluated with explicit round-to-nearest multiplies/adds (no FMA contraction), so for
// complex128 the result is bit-identical to the oracle (oracle/fgfrft_oracle.c) and
// Q(-alpha) = Q(alpha)^H holds bit-for-bit; integer orders give exact Kronecker results.
#include "common.cuh"

namespace fgb {

constexpr int kSynthStages = 4;    // TMA ring depth
constexpr int kSynthThreads = 256;

template <typename R>
__device__ __forceinline__ R rmul(R a, R b);
template <> __device__ __forceinline__ double rmul<double>(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ float rmul<float>(float a, float b) { return __fmul_rn(a, b); }
template <typename R>
__device__ __forceinline__ R radd(R a, R b);
template <> __device__ __forceinline__ double radd<double>(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ float radd<float>(float a, float b) { return __fadd_rn(a, b); }

// q += a*p + b*conj(pt), in the reference's evaluation order (no contraction).
template <typename R, typename C>
__device__ __forceinline__ void pair_update(C& q, R a, R b, const C& p, const C& pt) {
    q.x = radd<R>(q.x, radd<R>(rmul<R>(a, p.x), rmul<R>(b, pt.x)));
    q.y = radd<R>(q.y, radd<R>(rmul<R>(a, p.y), rmul<R>(b, -pt.y)));
}

size_t synth_smem_bytes(int elem_bytes, int l_used, int ac) {
    return (size_t)kSynthStages * 2 * kTileElems * elem_bytes + kSynthStages * 8 + (size_t)l_used * ac * 16 +
           (size_t)ac * 8 + 16;
}

// slabs: tiled layout (common.cuh), slab_elems = nt^2 * 1024 per power.
template <typename R, int AC>
__global__ void __launch_bounds__(kSynthThreads, 1)
synth_pairs_kernel(const cplx_t<R>* __restrict__ slabs, int n, int l_used, int64_t slab_elems,
                   const double* __restrict__ coef, int coef_ld, int lc, int n_alpha, int n_achunks,
                   cplx_t<R>* __restrict__ out, int64_t out_stride, int nt) {
    using C = cplx_t<R>;
    constexpr int T = kTile, S = kSynthStages;
    extern __shared__ __align__(128) unsigned char smem[];
    C* tiles = reinterpret_cast<C*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * 2 * kTileElems * sizeof(C));
    double2* cs = reinterpret_cast<double2*>(full + S);
    double* c0s = reinterpret_cast<double*>(cs + (size_t)l_used * AC);

    const int chunk = blockIdx.x % n_achunks;
    const int pair = blockIdx.x / n_achunks;
    int I, J;
    pair_of(pair, I, J);
    const int a0 = chunk * AC;
    const int na = min(AC, n_alpha - a0);
    const int bi = min(T, n - I * T), bj = min(T, n - J * T);
    const bool diag = (I == J);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int idx = tid; idx < l_used * AC; idx += kSynthThreads) {
        const int k = idx / AC + 1, a = idx % AC;
        double ak = 0.0, bk = 0.0;
        if (a < na) {
            const double* cr = coef + (size_t)(a0 + a) * coef_ld;
            ak = cr[lc + k];
            bk = cr[lc - k];
        }
        cs[idx] = make_double2(ak, bk);
    }
    if (tid < AC) c0s[tid] = tid < na ? coef[(size_t)(a0 + tid) * coef_ld + lc] : 0.0;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const uint32_t tile_bytes = (uint32_t)(kTileElems * sizeof(C));
    // Single order: the cache is streamed once, mark it evict-first. Several order chunks:
    // sibling CTAs of the same tile pair re-read it from L2, keep the default policy.
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
        for (int s = 0; s < S && s < l_used; ++s) issue(s + 1, s);

    const int r = lane;
    C q1[4][AC], q2[4][AC];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int c = warp + 8 * i;
#pragma unroll
        for (int a = 0; a < AC; ++a) {
            const R d = (diag && r == c) ? (R)c0s[a] : (R)0;
            q1[i][a].x = d;
            q1[i][a].y = 0;
            q2[i][a].x = 0;
            q2[i][a].y = 0;
        }
    }

    for (int k = 1; k <= l_used; ++k) {
        const int s = (k - 1) % S;
        mbar_wait(&full[s], ((k - 1) / S) & 1);
        const C* t1 = tiles + (size_t)(s * 2) * kTileElems;
        const C* t2 = diag ? t1 : t1 + kTileElems;
        double2 ab[AC];
#pragma unroll
        for (int a = 0; a < AC; ++a) ab[a] = cs[(k - 1) * AC + a];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = warp + 8 * i;
            const C p1 = t1[swz(r, c)];  // P[I*T + r, J*T + c]
            const C p2 = t2[swz(c, r)];  // P[J*T + c, I*T + r]
#pragma unroll
            for (int a = 0; a < AC; ++a) {
                pair_update<R>(q1[i][a], (R)ab[a].x, (R)ab[a].y, p1, p2);
                if (!diag) pair_update<R>(q2[i][a], (R)ab[a].x, (R)ab[a].y, p2, p1);
            }
        }
        __syncthreads();
        if (tid == 0 && k + S <= l_used) issue(k + S, s);
    }

    // Q[I,J]: lanes run down a column -> coalesced stores straight from registers.
#pragma unroll
    for (int a = 0; a < AC; ++a) {
        if (a >= na) break;
        C* o = out + (int64_t)(a0 + a) * out_stride;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = warp + 8 * i;
            if (r < bi && c < bj) o[(int64_t)(J * T + c) * n + I * T + r] = q1[i][a];
        }
    }
    if (diag) return;
    // Q[J,I]: transpose through shared memory (swizzled, conflict-free) so stores stay coalesced.
    C* buf = tiles;
#pragma unroll
    for (int a = 0; a < AC; ++a) {
        if (a >= na) break;
#pragma unroll
        for (int i = 0; i < 4; ++i) buf[swz(warp + 8 * i, r)] = q2[i][a];  // (row c, col r) of Q[J,I]
        __syncthreads();
        C* o = out + (int64_t)(a0 + a) * out_stride;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int col = warp + 8 * i;  // I-block column
            const int row = lane;          // J-block row
            if (row < bj && col < bi) o[(int64_t)(I * T + col) * n + J * T + row] = buf[swz(row, col)];
        }
        __syncthreads();
    }
}

// Host launcher. coef: device [n_alpha][2*l_used+1] (SincCoeffs layout with L = l_used).
template <typename R>
cudaError_t launch_synth(const void* slabs, int n, int l_used, const double* coef_dev, int n_alpha,
                         void* out, cudaStream_t stream) {
    const int nt = (int)ceil_div(n, kTile);
    const int npairs = nt * (nt + 1) / 2;
    const int ac = n_alpha >= 4 ? 4 : (n_alpha >= 2 ? 2 : 1);
    const int nchunks = (int)ceil_div(n_alpha, ac);
    const size_t smem = synth_smem_bytes(sizeof(cplx_t<R>), l_used, ac);
    const int64_t slab = (int64_t)nt * nt * kTileElems;
    const dim3 grid((unsigned)((int64_t)nchunks * npairs));
    const int coef_ld = 2 * l_used + 1;
#define FGB_SYNTH_CASE(ACV)                                                                                  \
    {                                                                                                        \
        auto kern = synth_pairs_kernel<R, ACV>;                                                              \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e != cudaSuccess) return e;                                                                      \
        kern<<<grid, kSynthThreads, smem, stream>>>((const cplx_t<R>*)slabs, n, l_used, slab, coef_dev,      \
                                                    coef_ld, l_used, n_alpha, nchunks, (cplx_t<R>*)out,      \
                                                    (int64_t)n * n, nt);                                     \
    }
    if (ac == 4) FGB_SYNTH_CASE(4) else if (ac == 2) FGB_SYNTH_CASE(2) else FGB_SYNTH_CASE(1)
#undef FGB_SYNTH_CASE
    return cudaGetLastError();
}

template cudaError_t launch_synth<double>(const void*, int, int, const double*, int, void*, cudaStream_t);
template cudaError_t launch_synth<float>(const void*, int, int, const double*, int, void*, cudaStream_t);

}  // namespace fgb
