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

// =====================================================================================
// Order sweeps on the FP64 tensor cores.
//
// For many orders the synthesis is the GEMM  Q[a][e] = sum_kk C[a][kk] V[kk][e]  with
// kk = (k, +/-): C = a_k(alpha) / b_k(alpha), V = P_k(e) / conj(P_k^T)(e). One CTA owns an 8x8
// sub-square of tile (I,J) plus its transposed partner in tile (J,I) (64 + 64 positions, e =
// position x re/im = 256 columns) for up to 64 orders (rows), and streams the cached powers at
// those positions (each cache element is staged by exactly one CTA, so the cache crosses HBM
// once per launch, not once per order chunk). 8 warps: warp w owns the 32 e-columns
// [32w, 32w+32) for all 64 orders: per K4 step 8 coefficient fragments + 4 cache fragments feed
// 32 DMMAs. Coefficients are staged per chunk of 64 powers ([a][kk], padded), cache values
// through a 3-stage cp.async ring of 8 powers; outputs leave through shared memory so stores
// are 128-byte runs. Rounding differs from the exact scalar path (DMMA accumulation): the result
// matches it to ~1e-16 relative instead of bit-for-bit.
// =====================================================================================

constexpr int kSwA = 64, kSwKc = 64, kSwStK = 8, kSwStages = 3;
constexpr int kSwCLd = 2 * kSwKc + 4;  // doubles per coefficient row
constexpr int kSwPLd = 66;             // complex per (power, tile) staging row

size_t synth_sweep_smem_bytes() {
    const size_t cs = (size_t)kSwA * kSwCLd * 8;
    const size_t st = (size_t)kSwStages * kSwStK * 2 * kSwPLd * 16;
    const size_t os = (size_t)kSwA * 66 * 16;
    return (cs + st) > os ? cs + st : os;
}

__global__ void __launch_bounds__(256, 1)
synth_sweep_mma_kernel(const double2* __restrict__ slabs, int n, int l_used, int64_t slab_elems,
                       const double* __restrict__ coef, int coef_ld, int lc, int n_alpha,
                       double2* __restrict__ out, int64_t out_stride, int nt) {
    extern __shared__ __align__(128) unsigned char smem[];
    double* cs = reinterpret_cast<double*>(smem);
    double2* stb = reinterpret_cast<double2*>(smem + (size_t)kSwA * kSwCLd * 8);
    double2* os = reinterpret_cast<double2*>(smem);  // epilogue reuse

    const int pair = blockIdx.x >> 4, sq = blockIdx.x & 15;
    int I, J;
    pair_of(pair, I, J);
    const bool diag = (I == J);
    const int sr = sq & 3, sc = sq >> 2;
    if (diag && sr > sc) return;  // covered by the transposed sub-square
    const int r0 = 8 * sr, c0 = 8 * sc;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int tw = warp >> 2, pbase = 16 * (warp & 3);
    const int64_t b1 = tile_base(I, J, nt), b2 = tile_base(J, I, nt);

    double d[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) d[i][j][0] = d[i][j][1] = 0.0;

    for (int k0 = 1; k0 <= l_used; k0 += kSwKc) {
        const int kc = min(kSwKc, l_used - k0 + 1);
        const int nsteps = (kc + kSwStK - 1) / kSwStK;
        __syncthreads();  // previous chunk finished with cs / stb
        for (int idx = tid; idx < kSwA * 2 * kSwKc; idx += 256) {
            const int a = idx / (2 * kSwKc), kk = idx % (2 * kSwKc);
            const int k = k0 + (kk >> 1);
            double v = 0.0;
            if (a < n_alpha && (kk >> 1) < kc) v = coef[(size_t)a * coef_ld + lc + ((kk & 1) ? -k : k)];
            cs[a * kSwCLd + kk] = v;
        }
        // stage st: powers k0 + 8 st + kp at the 64 + 64 positions (p = jj*8 + ii)
        auto stage = [&](int st, int buf) {
            double2* dst0 = stb + (size_t)buf * kSwStK * 2 * kSwPLd;
            for (int idx = tid; idx < kSwStK * 2 * 64; idx += 256) {
                const int kp = idx >> 7, t = (idx >> 6) & 1, p = idx & 63;
                const int ii = p & 7, jj = p >> 3;
                const int kq = 8 * st + kp;
                const bool v = kq < kc;
                const double2* slab = slabs + (int64_t)(k0 + (v ? kq : 0) - 1) * slab_elems;
                const double2* src = t == 0 ? slab + b1 + swz(r0 + ii, c0 + jj) : slab + b2 + swz(c0 + jj, r0 + ii);
                cp_async16(dst0 + (kp * 2 + t) * kSwPLd + p, src, v);
            }
        };
#pragma unroll
        for (int s = 0; s < kSwStages - 1; ++s) {
            if (s < nsteps) stage(s, s);
            cp_async_commit();
        }
        for (int st = 0; st < nsteps; ++st) {
            cp_async_wait<kSwStages - 2>();
            __syncthreads();
            if (st + kSwStages - 1 < nsteps) stage(st + kSwStages - 1, (st + kSwStages - 1) % kSwStages);
            cp_async_commit();
            const double* sb = reinterpret_cast<const double*>(stb + (size_t)(st % kSwStages) * kSwStK * 2 * kSwPLd);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const int kkl = 4 * ks + t4;          // power term within the stage
                const int kp = kkl >> 1, sign = kkl & 1;
                double b[4];
                const int tt = sign ? 1 - tw : tw;
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) {
                    const int p = pbase + 4 * nb + (g >> 1), comp = g & 1;
                    const double v = sb[((kp * 2 + tt) * kSwPLd + p) * 2 + comp];
                    b[nb] = (sign && comp) ? -v : v;
                }
                const double* crow = cs + g * kSwCLd + 16 * st + kkl;
#pragma unroll
                for (int mb = 0; mb < 8; ++mb) {
                    const double a = crow[8 * mb * kSwCLd];
#pragma unroll
                    for (int nb = 0; nb < 4; ++nb) dmma884(d[mb][nb][0], d[mb][nb][1], a, b[nb]);
                }
            }
        }
    }
    cp_async_wait<0>();

    // Epilogue: identity term c_0 on the global diagonal, then coalesced stores via smem.
    for (int t = 0; t < 2; ++t) {
        if (t == 1 && diag && sr == sc) break;
        __syncthreads();
        if (tw == t) {
#pragma unroll
            for (int mb = 0; mb < 8; ++mb)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb) {
                    const int a = 8 * mb + g;
                    const int p = pbase + 4 * nb + t4;
                    const int ii = p & 7, jj = p >> 3;
                    double re = d[mb][nb][0];
                    if (t == 0 && diag && sr == sc && ii == jj && a < n_alpha)
                        re += coef[(size_t)a * coef_ld + lc];
                    // t = 0: column-major over (ii fast); t = 1: transposed so writes stay contiguous
                    const int q = t == 0 ? p : ii * 8 + jj;
                    os[a * 66 + q] = make_double2(re, d[mb][nb][1]);
                }
        }
        __syncthreads();
        for (int idx = tid; idx < kSwA * 64; idx += 256) {
            const int a = idx >> 6, q = idx & 63;
            if (a >= n_alpha) break;
            const int hi = q >> 3, lo = q & 7;
            int row, col;
            if (t == 0) {  // q = jj*8 + ii: rows r0+ii of column c0+jj in tile (I,J)
                row = I * 32 + r0 + lo;
                col = J * 32 + c0 + hi;
            } else {       // q = ii*8 + jj: rows c0+jj of column r0+ii in tile (J,I)
                row = J * 32 + c0 + lo;
                col = I * 32 + r0 + hi;
            }
            if (row < n && col < n) out[(int64_t)a * out_stride + (int64_t)col * n + row] = os[a * 66 + q];
        }
    }
}

int synth_sweep_max_orders() { return kSwA; }

// n_alpha <= 64. coef: device [n_alpha][2*l_used+1].
cudaError_t launch_synth_sweep(const void* slabs, int n, int l_used, const double* coef_dev, int n_alpha, void* out,
                               cudaStream_t stream) {
    const int nt = (int)ceil_div(n, kTile);
    const int npairs = nt * (nt + 1) / 2;
    const size_t smem = synth_sweep_smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(synth_sweep_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    synth_sweep_mma_kernel<<<(unsigned)npairs * 16, 256, smem, stream>>>(
        (const double2*)slabs, n, l_used, (int64_t)nt * nt * kTileElems, coef_dev, 2 * l_used + 1, l_used, n_alpha,
        (double2*)out, (int64_t)n * n, nt);
    return cudaGetLastError();
}

}  // namespace fgb
