// packed.cu -- the packed power cache and its synthesis kernel (the one- / two-order step route).
//
// The MSE step and the series apply of one or two orders are bound by streaming the L cached
// powers once (transform.hpp:111-136: every call reads every slab). For a real F (every
// BASELINE graph) the step route keeps, next to the exact FP64 slabs (which fgfrft_matrix /
// fgfrft_grad still read, bit-exactly), a PACKED copy: each 32x32 tile of each power as 40-bit
// fixed-point mantissas relative to a per-tile power of two,
//     P_k[i, j] = m * 2^(e_kT - 38),  |m| <= 2^38,  max_T |P_k| < 2^e_kT,
// stored as a 32-bit low plane and an 8-bit high plane of u = m + 2^39 (5 bytes per element
// instead of 8: 37.5% fewer bytes on the HBM-bound pass). Decoding is exact integer arithmetic:
// the double with high word 0x43300000 | hi and low word lo is 2^52 + u, so m = that - (2^52 +
// 2^39) with no rounding; the tile scale is folded into the series coefficient (a power-of-two
// product, exact), so each element costs one DADD and two DFMAs per order. Quantisation error:
// <= 2^-39 of the tile's largest |entry| per element (a few 1e-12 relative on Q, measured in
// tests/test_gpu_packed.py): inside the 1e-10 relative Frobenius parity bar; the
// exact path (fgfrft_matrix / fgfrft_grad) is untouched.
//
// psynth_pairs_kernel mirrors rsynth_pairs_kernel (real.cu): one CTA per tile pair {(I,J),(J,I)},
// a TMA bulk-copy ring of packed tiles, both tiles of Q updated from the same staged bytes. It
// also leaves the row maxima |Q[i, :]| (as ordered double bits, atomicMax) that the Ozaki
// slicing of Q for the product GEMM needs, so Q is read once by the slicer instead of twice.
#include "common.cuh"

namespace fgb {

constexpr int kPkTileBytes = kTileElems * 5;  // lo32 plane (4096 B) + hi8 plane (1024 B)
constexpr int kPkFrac = 38;
__device__ constexpr double kPkMagic = 4503599627370496.0 + 549755813888.0;  // 2^52 + 2^39

size_t packed_bytes(int n, int l) {  // pair-major records: npairs * L * 2 tiles
    const int64_t nt = ceil_div(n, kTile);
    return (size_t)(nt * (nt + 1) / 2) * (size_t)l * 2 * kPkTileBytes;
}
size_t packed_scale_elems(int n, int l) {
    const int64_t nt = ceil_div(n, kTile);
    return (size_t)(nt * (nt + 1) / 2) * (size_t)l * 2;
}

// One CTA per tile of every power: grid = l * ntiles, 256 threads x 4 elements.
// Pair-major layout: tile pair p = {(I,J), (J,I)} (I-major order, pairs_before below), power k:
// both tiles in one 10 KB record at ((p * L + k - 1) * 2 + slot) * 5120 bytes, slot 0 = (I,J),
// slot 1 = (J,I) (a diagonal tile is stored in both slots), scales at (p * L + k - 1) * 2 + slot.
// A CTA walking a pair streams one contiguous L * 10 KB region, one bulk copy per power.

// One CTA per tile of every power: grid = l * ntiles, 256 threads x 4 elements.
// pmax (optional, [L][2][32 nt] ordered double bits, zeroed by the caller): max_j |P_k[i, j]| (slot 0)
// and max_j |P_k[j, i]| (slot 1) of every power, plus the tile's quantum (so they bound the DECODED
// values) -- the per-row bounds the digit-emitting synthesis scales Q's rows by (prow_bound_kernel).
__global__ void __launch_bounds__(256) pack_tiles_kernel(const double* __restrict__ slabs, int64_t slab_elems,
                                                         int nt, int l, unsigned char* __restrict__ packed,
                                                         double* __restrict__ scales,
                                                         unsigned long long* __restrict__ pmax) {
    __shared__ double red[8];
    __shared__ double ab[kTile][kTile + 1];
    const int64_t ntiles = (int64_t)nt * nt;
    const int64_t tile = blockIdx.x;
    const int64_t k = tile / ntiles, t = tile - k * ntiles;  // k = power - 1; t = J * nt + I
    const int I = (int)(t % nt), J = (int)(t / nt);
    const double* src = slabs + k * slab_elems + t * kTileElems;
    double v[4];
    double m = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        v[i] = src[threadIdx.x + 256 * i];
        m = fmax(m, fabs(v[i]));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    double mx = red[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) mx = fmax(mx, red[w]);
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
    e = max(e, -900);              // all-tiny tiles quantise to 0 instead of overflowing the scale
    const double up = ldexp(1.0, kPkFrac - e);
    if (pmax) {  // element t = (row (t & 31) ^ (t >> 5), column t >> 5) of the swizzled tile
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int t = threadIdx.x + 256 * i, cj = t >> 5;
            ab[(t & 31) ^ cj][cj] = fabs(v[i]);
        }
        __syncthreads();
        if (threadIdx.x < 2 * kTile) {
            const int q = threadIdx.x & 31, col = threadIdx.x >> 5;  // col 0: row q's max, 1: column q's
            double m2 = 0.0;
            for (int z = 0; z < kTile; ++z) m2 = fmax(m2, col ? ab[z][q] : ab[q][z]);
            m2 += ldexp(1.0, e - kPkFrac);  // the decoded value is within one quantum
            const int64_t npad = (int64_t)nt * kTile;
            atomicMax(pmax + (k * 2 + col) * npad + (col ? J : I) * kTile + q,
                      (unsigned long long)__double_as_longlong(m2));
        }
    }
    const int lo_i = min(I, J), hi_j = max(I, J);
    const int64_t pair = pairs_before(lo_i, nt) + (hi_j - lo_i);
    for (int slot = (I <= J ? 0 : 1); slot <= (I < J ? 0 : 1); ++slot) {  // diagonal: both slots
        const int64_t rec = (pair * l + k) * 2 + slot;
        unsigned char* dst = packed + rec * kPkTileBytes;
        uint32_t* lo = reinterpret_cast<uint32_t*>(dst);
        uint8_t* hi = dst + kTileElems * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const long long mi = __double2ll_rn(v[i] * up);  // |mi| <= 2^38
            const unsigned long long u = (unsigned long long)(mi + (1LL << 39));
            lo[threadIdx.x + 256 * i] = (uint32_t)u;
            hi[threadIdx.x + 256 * i] = (uint8_t)(u >> 32);
        }
        if (threadIdx.x == 0) scales[rec] = ldexp(1.0, e - kPkFrac);
    }
}

cudaError_t launch_pack_tiles(const void* slabs, int n, int l, void* packed, double* scales, cudaStream_t stream,
                              unsigned long long* pmax) {
    const int nt = (int)ceil_div(n, kTile);
    const int64_t ntiles = (int64_t)nt * nt;
    if (pmax) {
        cudaError_t e = cudaMemsetAsync(pmax, 0, (size_t)l * 2 * nt * kTile * sizeof(unsigned long long), stream);
        if (e != cudaSuccess) return e;
    }
    pack_tiles_kernel<<<(unsigned)(ntiles * l), 256, 0, stream>>>((const double*)slabs, ntiles * kTileElems, nt, l,
                                                                  (unsigned char*)packed, scales, pmax);
    return cudaGetLastError();
}

// Row bounds of Q_a - c_0 I from the power maxima: R_i = sum_(k=1..l) |c_a(k)| max_j |P_k[i, j]| +
// |c_a(-k)| max_j |P_k[j, i]| >= max_j |Q_a[i, j] - c_0 delta_ij| (the series' triangle inequality;
// inflated by 2^-40 for the synthesis' own FP64 rounding), and exps[a rp + i] = e with R_i < 2^e --
// the row exponents of the product GEMM's Ozaki slicing (|Q[i, :]| 2^(-e-1) < 1/2), known BEFORE
// Q exists, so the synthesis can emit Q's digits directly (psynth_pairs_kernel SD > 0). A row whose
// bound is loose by 2^b loses b bits of the ~47 the 6 digits carry (measured ~2.5 bits on graph
// GFTs: 4-6x at N = 1024). coef rows: a * coef_ld, c_k at l + k.
// 64 rows x 4 power slices per CTA (k = 1 + slice, 5 + slice, ...; the slices' partial sums are added
// in fixed order through shared memory): the kernel sits on the step's critical path ahead of the
// synthesis, so it is spread over rp / 64 CTAs instead of one serial 2 l-load chain per thread.
__global__ void __launch_bounds__(256) prow_bound_kernel(const unsigned long long* __restrict__ pmax, int64_t npad,
                                                         int l, const double* __restrict__ coef, int coef_ld, int rp,
                                                         int* __restrict__ exps) {
    __shared__ double part[4][64];
    const int lr = threadIdx.x & 63, ks = threadIdx.x >> 6;
    const int i = blockIdx.x * 64 + lr, a = blockIdx.y;
    const double* cr = coef + (int64_t)a * coef_ld + l;
    double r = 0.0;
    if (i < npad && i < rp) {
#pragma unroll 4
        for (int k = 1 + ks; k <= l; k += 4) {
            const double mr = __longlong_as_double((long long)pmax[(int64_t)(k - 1) * 2 * npad + i]);
            const double mc = __longlong_as_double((long long)pmax[((int64_t)(k - 1) * 2 + 1) * npad + i]);
            r = fma(fabs(cr[k]), mr, fma(fabs(cr[-k]), mc, r));
        }
    }
    part[ks][lr] = r;
    __syncthreads();
    if (ks != 0 || i >= rp) return;
    r = ((part[0][lr] + part[1][lr]) + part[2][lr]) + part[3][lr];
    r *= 1.0 + 0x1p-40;
    int e = 0;
    if (r > 0.0) frexp(r, &e);
    exps[(int64_t)a * rp + i] = e;
}

cudaError_t launch_prow_bound(const unsigned long long* pmax, int n, int l, const double* coef, int coef_ld, int ac,
                              int rp, int* exps, cudaStream_t stream) {
    const int64_t npad = ceil_div(n, kTile) * kTile;
    prow_bound_kernel<<<dim3((unsigned)ceil_div(rp, 64), (unsigned)ac), 256, 0, stream>>>(pmax, npad, l, coef,
                                                                                         coef_ld, rp, exps);
    return cudaGetLastError();
}

int64_t packed_pairs_before(int I, int nt) { return pairs_before(I, nt); }


// Persistent form: 2 CTAs per SM, each walking its pairs p0 + blockIdx.x + j * gridDim.x. A
// dedicated producer warp keeps a TMA ring of (pair, power) items full ACROSS pairs (consumer
// warps release stages through `empty` mbarriers, no CTA-wide barrier per power), so the next
// pair's tiles stream in while this pair's epilogue (stores, row maxima) runs; the per-tile
// scales of a pair arrive by bulk copy into a double buffer. Decode + scale is one exact DFMA
// (d s - (2^52 + 2^39) s, s a power of two); the series coefficients are a table shared by all pairs.
constexpr int kPsStages = 10;
constexpr int kPsConsumers = 256;


// G independent producer / consumer groups per CTA (one CTA per SM): each group has its own ring,
// barriers, scale buffers and tables, and walks its own pairs; a capped grid therefore occupies
// exactly that many SMs and leaves the others whole for a concurrent GEMM (the shell pipeline).
__host__ __device__ __forceinline__ size_t psynth_group_bytes(int l, int ac, int stages = kPsStages) {
    const size_t b = (size_t)stages * 2 * kPkTileBytes + (2 * stages + 2) * 8 + (size_t)2 * 2 * l * 8 +
                     (size_t)ac * (2 * l + 1) * 8 + (size_t)ac * 8 * 32 * 8;
    return (b + 127) & ~(size_t)127;
}
static int psynth_groups(int ac) { return ac == 4 ? 1 : 2; }
size_t psynth_smem_bytes(int l, int ac, int stages) { return psynth_groups(ac) * psynth_group_bytes(l, ac, stages); }
static int psynth_stages(int l, int ac) {  // the deepest ring that fits 227 KB (10 or 8 stages)
    return psynth_smem_bytes(l, ac, kPsStages) <= 227 * 1024 ? kPsStages : 8;
}

__device__ __forceinline__ void consumer_sync(int g) { asm volatile("bar.sync %0, 256;" ::"r"(1 + g) : "memory"); }

// Stage s of a pair's items is (k - 1) % S (every pair restarts at stage 0, so the consumer's
// stage offsets are compile-time immediates); per-stage phase bits track the reuse.
// SD > 0 (digit emission, n % 128 == 0): instead of FP64 Q and its row maxima, the kernel writes Q's
// SD balanced base-254 digits straight into the product GEMM's sliced A operand (ozgemm.cu layout:
// 128-row tiles x 64-byte K blocks, SD digit planes of 8 KB per block, 8-row core groups 512 B apart),
// scaled per row by the exponents prow_bound_kernel derived from the power maxima -- the FP64 Q round
// trip through HBM and the slicing pass disappear. Digit arithmetic = oz_write_digits'.
struct PsDigits {
    int8_t* dig = nullptr;
    const int* exps = nullptr;  // [a * rp + row]
    int rp = 0, kbc = 0;        // padded rows per output block, 64-byte K blocks
};

template <int SD>
__device__ __forceinline__ void ps_digits4(double (&x)[4], int8_t* base) {  // 4 consecutive K of one row
#pragma unroll
    for (int s = 0; s < SD; ++s) {
        uint32_t w = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double y = x[i] * 254.0;
            const double t = y + 6755399441055744.0;  // rint(y) in the low word
            x[i] = y - (t - 6755399441055744.0);
            w |= ((uint32_t)__double2loint(t) & 0xFFu) << (8 * i);
        }
        *reinterpret_cast<uint32_t*>(base + s * 8192) = w;
    }
}
template <int SD>
__device__ __forceinline__ void ps_digits1(double x, int8_t* base) {
#pragma unroll
    for (int s = 0; s < SD; ++s) {
        const double y = x * 254.0;
        const double t = y + 6755399441055744.0;
        x = y - (t - 6755399441055744.0);
        base[s * 8192] = (int8_t)__double2loint(t);
    }
}
__device__ __forceinline__ int8_t* ps_digit_addr(int8_t* dig, int sd, int kbc, int m, int k) {
    return dig + ((int64_t)(m >> 7) * kbc + (k >> 6)) * (sd * 8192) + ((m & 127) >> 3) * 512 + ((k >> 4) & 3) * 128 +
           (m & 7) * 16 + (k & 15);
}

template <int AC, int G, int S, int SD = 0>
__global__ void __launch_bounds__(G * (kPsConsumers + 32), 1)
psynth_pairs_kernel(const unsigned char* __restrict__ packed, const double* __restrict__ scales, int n, int l,
                    int lc, const double* __restrict__ coef, int coef_ld, double* __restrict__ out, int64_t out_stride,
                    unsigned long long* __restrict__ rowmax, int64_t rm_stride, int nt, int p0, int p1,
                    int pbase, int nodiag, PsDigits pd) {
    constexpr int kStage = 2 * kPkTileBytes;
    extern __shared__ __align__(128) unsigned char smem_all[];
    const int g = threadIdx.x / (kPsConsumers + 32);
    unsigned char* smem = smem_all + (size_t)g * psynth_group_bytes(lc, AC, S);
    unsigned char* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * kStage);
    uint64_t* empty = full + S;
    uint64_t* sbar = empty + S;                                          // [2] scale buffers
    double* sbuf = reinterpret_cast<double*>(sbar + 2);                  // [2][lc][2]
    double* ctab = sbuf + 4 * lc;                                        // [AC][2l + 1]
    double* red = ctab + AC * (2 * l + 1);                               // [AC][8][32]
    const int tid = threadIdx.x - g * (kPsConsumers + 32), lane = tid & 31, warp = tid >> 5;
    const int vcta = (int)blockIdx.x * G + g, vgrid = (int)gridDim.x * G;  // this group's pairs
    const int npairs = (p1 - p0 - vcta + vgrid - 1) / vgrid;
    const int depth = S < l ? S : l;  // stages in use; <= l, so a pair's scale buffer is never refilled in use
    const int cw = 2 * l + 1;
    // nodiag: Q - c_0 I (the product GEMM adds c_0 X in its epilogue, so Q's row maxima -- and the
    // Ozaki slicing error -- follow the off-diagonal entries)
    for (int idx = tid; idx < AC * cw; idx += kPsConsumers + 32)
        ctab[idx] = (nodiag && idx % cw == l) ? 0.0 : coef[(size_t)(idx / cw) * coef_ld + idx % cw];
    if (tid == 0) {
        for (int q = 0; q < S; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], kPsConsumers / 32);
        }
        mbar_init(&sbar[0], 1);
        mbar_init(&sbar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (npairs <= 0) return;
    if (warp == kPsConsumers / 32) {  // ---------------- producer warp (one elected lane)
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            uint32_t used = 0, eph = 0;
            for (int j = 0; j < npairs; ++j) {
                const int64_t pr = p0 + vcta + (int64_t)j * vgrid - pbase;  // local record index
                const unsigned char* src = packed + pr * lc * kStage;       // this pair's contiguous records
                int q = 0;
                for (int k = 1; k <= l; ++k) {
                    if (used >> q & 1) {
                        mbar_wait(&empty[q], eph >> q & 1);
                        eph ^= 1u << q;
                    }
                    used |= 1u << q;
                    if (k == 1) {  // the pair's tile scales, both tiles, all powers
                        mbar_arrive_expect_tx(&sbar[j & 1], 2 * lc * 8);
                        bulk_g2s(sbuf + (size_t)(j & 1) * 2 * lc, scales + pr * lc * 2, 2 * lc * 8, &sbar[j & 1]);
                    }
                    mbar_arrive_expect_tx(&full[q], kStage);
                    bulk_g2s_hint(ring + (size_t)q * kStage, src + (int64_t)(k - 1) * kStage, kStage, &full[q], pol);
                    if (++q == depth) q = 0;
                }
            }
        }
        return;
    }
    // ---------------- consumer warps: thread (lane r, warp) owns elements (r, c_i) of tile (I,J)
    // and (c_i, r) of tile (J,I), c_i = 4 warp + i (4 consecutive K of a row: one 32-bit digit store
    // per digit plane when emitting); their byte offsets inside a stage are fixed (the XOR swizzle
    // keeps every fixed-c_i read conflict free)
    const int r = lane;
    const uint32_t* lo1p[4];  // element (r, c_i) of tile 1 and (c_i, r) of tile 2, stage 0
    const uint8_t* hi1p[4];
    const uint32_t* lo2p[4];
    const uint8_t* hi2p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int c = 4 * warp + i;
        lo1p[i] = reinterpret_cast<const uint32_t*>(ring) + swz(r, c);
        hi1p[i] = ring + kTileElems * 4 + swz(r, c);
        lo2p[i] = reinterpret_cast<const uint32_t*>(ring + kPkTileBytes) + swz(c, r);
        hi2p[i] = ring + kPkTileBytes + kTileElems * 4 + swz(c, r);
    }
    uint32_t fph = 0;
    for (int j = 0; j < npairs; ++j) {
        int I, J;
        pair_of_imajor(p0 + vcta + j * vgrid, nt, I, J);
        const bool diag = I == J;
        const int bi = min(kTile, n - I * kTile), bj = min(kTile, n - J * kTile);
        mbar_wait(&sbar[j & 1], (j >> 1) & 1);
        const double* sv = sbuf + (size_t)(j & 1) * 2 * lc;  // [k][slot]
        double q1[4][AC], q2[4][AC];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int a = 0; a < AC; ++a) {
                q1[i][a] = (diag && r == 4 * warp + i) ? ctab[a * cw + l] : 0.0;
                q2[i][a] = 0.0;
            }
        for (int k0 = 1; k0 <= l; k0 += S) {
#pragma unroll
            for (int u = 0; u < S; ++u) {
                const int k = k0 + u;
                if (k > l) break;
                mbar_wait(&full[u], fph >> u & 1);
                fph ^= 1u << u;
                const double sc1 = sv[2 * (k - 1)], sc2 = sv[2 * (k - 1) + 1];
                const double ns1 = -kPkMagic * sc1, ns2 = -kPkMagic * sc2;  // exact (powers of two)
                double ck[AC], cm[AC];
#pragma unroll
                for (int a = 0; a < AC; ++a) {
                    ck[a] = ctab[a * cw + l + k];
                    cm[a] = ctab[a * cw + l - k];
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    // stage offsets are immediates (u is unrolled): LDS [R + imm], no address math
                    const uint32_t lo1 = lo1p[i][u * (kStage / 4)], hi1 = hi1p[i][u * kStage];
                    const uint32_t lo2 = lo2p[i][u * (kStage / 4)], hi2 = hi2p[i][u * kStage];
                    // (2^52 + u) s - (2^52 + 2^39) s = m s exactly: one rounding-free FMA per value
                    const double p1 = fma(__hiloint2double((int)(0x43300000u | hi1), (int)lo1), sc1, ns1);
                    const double p2 = fma(__hiloint2double((int)(0x43300000u | hi2), (int)lo2), sc2, ns2);
#pragma unroll
                    for (int a = 0; a < AC; ++a) {
                        q1[i][a] = fma(ck[a], p1, fma(cm[a], p2, q1[i][a]));
                        q2[i][a] = fma(ck[a], p2, fma(cm[a], p1, q2[i][a]));  // unused on diagonal pairs
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[u]);
            }
        }
        if constexpr (SD > 0) {  // digits of both tiles straight into the product GEMM's A operand
#pragma unroll
            for (int a = 0; a < AC; ++a) {
                {  // Q[32 I + r, 32 J + 4 warp .. + 3]: one 32-bit store per digit plane
                    const int m = a * pd.rp + I * kTile + r, k0 = J * kTile + 4 * warp;
                    const double sc = __longlong_as_double((long long)(1022 - pd.exps[m]) << 52);  // 2^(-e-1)
                    double x[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) x[i] = q1[i][a] * sc;
                    ps_digits4<SD>(x, ps_digit_addr(pd.dig, SD, pd.kbc, m, k0));
                }
                if (!diag) {  // Q[32 J + 4 warp + i, 32 I + r]: lanes along K, byte stores
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int m = a * pd.rp + J * kTile + 4 * warp + i;
                        const double sc = __longlong_as_double((long long)(1022 - pd.exps[m]) << 52);
                        ps_digits1<SD>(q2[i][a] * sc, ps_digit_addr(pd.dig, SD, pd.kbc, m, I * kTile + r));
                    }
                }
            }
        } else {
        // Q[I-tile, J-tile]: rows r (lanes), columns c = 4 warp + i; row maxima across the 8 warps
#pragma unroll
        for (int a = 0; a < AC; ++a) {
            double mx = 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int c = 4 * warp + i;
                if (r < bi && c < bj) {
                    out[(int64_t)a * out_stride + (int64_t)(J * kTile + c) * n + I * kTile + r] = q1[i][a];
                    mx = fmax(mx, fabs(q1[i][a]));
                }
            }
            red[(a * 8 + warp) * 32 + lane] = mx;
        }
        if (!diag) {
            // Q[J-tile, I-tile]: thread (lane r, warp) holds Q[J*32 + 4 warp + i, I*32 + r]
#pragma unroll
            for (int a = 0; a < AC; ++a)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int row = 4 * warp + i;
                    const bool ok = r < bi && row < bj;
                    double m = ok ? fabs(q2[i][a]) : 0.0;
                    if (ok) out[(int64_t)a * out_stride + (int64_t)(I * kTile + r) * n + J * kTile + row] = q2[i][a];
#pragma unroll
                    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
                    if (lane == 0 && row < bj && m > 0.0)
                        atomicMax(rowmax + (int64_t)a * rm_stride + J * kTile + row,
                                  (unsigned long long)__double_as_longlong(m));
                }
        }
        consumer_sync(g);
        if (warp < AC) {
            const int a = warp;
            double mx = red[(a * 8) * 32 + lane];
#pragma unroll
            for (int w = 1; w < 8; ++w) mx = fmax(mx, red[(a * 8 + w) * 32 + lane]);
            if (r < bi && mx > 0.0)
                atomicMax(rowmax + (int64_t)a * rm_stride + I * kTile + r, (unsigned long long)__double_as_longlong(mx));
        }
        consumer_sync(g);
        }  // SD == 0
    }
}

// Tile pairs [p0, p1) of the I-major enumeration (p1 < 0: all of them); max_ctas > 0 caps the
// persistent grid.
// l: powers summed (the truncation), l_cache: powers stored (the scale layout's stride).
cudaError_t launch_psynth(const void* packed, const double* scales, int n, int l, int l_cache, const double* coef_dev,
                          int coef_ld, int n_alpha, double* out, int64_t out_stride, unsigned long long* rowmax,
                          int64_t rm_stride, cudaStream_t stream, int p0, int p1, int max_ctas, int pbase,
                          int nodiag, int8_t* digits, const int* exps, int rp, int kp, int sd) {
    const int nt = (int)ceil_div(n, kTile);
    if (p1 < 0) p1 = nt * (nt + 1) / 2;
    const int npairs = p1 - p0;
    if (npairs <= 0) return cudaSuccess;
    // digit emission: one order's [Q; dQ] (AC = 2), whole 128-row tiles, 5 / 6 digits
    if (digits && (n_alpha != 2 || n % 128 || rp % 128 || kp % 64 || (sd != 5 && sd != 6) || !exps))
        return cudaErrorInvalidValue;
    PsDigits pd;
    if (digits) {
        pd.dig = digits;
        pd.exps = exps;
        pd.rp = rp;
        pd.kbc = kp / 64;
    }
    const int stages = psynth_stages(l_cache, n_alpha);
    const size_t smem = psynth_smem_bytes(l_cache, n_alpha, stages);
    const int groups = psynth_groups(n_alpha);
    int grid = FGFRFT_SMS;  // one CTA (groups x 288 threads) per SM
    if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
    if (grid * groups > npairs) grid = (npairs + groups - 1) / groups;
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
#define FGB_PS(ACV, SDV)                                                                                     \
    {                                                                                                        \
        constexpr int GV = ACV == 4 ? 1 : 2;                                                                 \
        static PerDeviceOnce attr;                                                                           \
        cudaError_t e = attr.run([] {                                                                        \
            cudaError_t r = cudaFuncSetAttribute(psynth_pairs_kernel<ACV, GV, kPsStages, SDV>,               \
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);   \
            if (r != cudaSuccess) return r;                                                                  \
            return cudaFuncSetAttribute(psynth_pairs_kernel<ACV, GV, 8, SDV>,                                \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);            \
        });                                                                                                  \
        if (e != cudaSuccess) return e;                                                                      \
        auto kern = stages == kPsStages ? psynth_pairs_kernel<ACV, GV, kPsStages, SDV>                       \
                                        : psynth_pairs_kernel<ACV, GV, 8, SDV>;                              \
        kern<<<grid, GV * (kPsConsumers + 32), smem, stream>>>((const unsigned char*)packed,                 \
                                                              scales, n, l, l_cache,                         \
                                                              coef_dev, coef_ld, out, out_stride, rowmax,    \
                                                              rm_stride, nt, p0, p1, pbase, nodiag, pd);     \
    }
    if (digits) {
        if (sd == 6) FGB_PS(2, 6) else FGB_PS(2, 5)
    } else if (n_alpha == 1) FGB_PS(1, 0) else if (n_alpha == 2) FGB_PS(2, 0) else if (n_alpha == 4) FGB_PS(4, 0)
    else return cudaErrorInvalidValue;
#undef FGB_PS
    return cudaGetLastError();
}

// Pair-sharded build (capi_pshard.cu): rank g owns the pairs whose smaller tile index lies in
// [I0, I1) and never holds the full cache. Per power k it keeps the row panel P_k[R, :] and the
// column panel P_k[:, R] (R = rows [32 I0, 32 I1), real, column-major, ld_r = |R|, ld_c = n) and
// packs its pairs' records for that power from them: slot 0 = tile (I, J) from the row panel,
// slot 1 = tile (J, I) from the column panel. Records are local: index (pair - pbase).
__global__ void __launch_bounds__(256) pack_pairs_from_panels_kernel(const double* __restrict__ rp, int64_t ld_r,
                                                                     const double* __restrict__ cp, int64_t ld_c,
                                                                     int n, int nt, int I0, int pbase, int k, int l,
                                                                     unsigned char* __restrict__ packed,
                                                                     double* __restrict__ scales) {
    __shared__ double red[8];
    const int local = (int)(blockIdx.x >> 1), slot = (int)(blockIdx.x & 1);
    int I, J;
    pair_of_imajor(pbase + local, nt, I, J);
    const int r0 = I0 * kTile;
    double v[4];
    double m = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int t = threadIdx.x + 256 * q;            // tile position t = j * 32 + (i ^ j)
        const int jj = t >> 5, ii = (t & 31) ^ jj;      // element (ii, jj) of the tile
        double x = 0.0;
        if (slot == 0) {                                 // tile (I, J): rows I*32 + ii of the row panel
            const int gr = I * kTile + ii, gc = J * kTile + jj;
            if (gr < n && gc < n) x = rp[(int64_t)(gr - r0) + (int64_t)gc * ld_r];
        } else {                                         // tile (J, I): columns I*32 + jj of the column panel
            const int gr = J * kTile + ii, gc = I * kTile + jj;
            if (gr < n && gc < n) x = cp[(int64_t)gr + (int64_t)(gc - r0) * ld_c];
        }
        v[q] = x;
        m = fmax(m, fabs(x));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    double mx = red[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) mx = fmax(mx, red[w]);
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);
    e = max(e, -900);
    const double up = ldexp(1.0, kPkFrac - e);
    const int64_t rec = ((int64_t)local * l + k) * 2 + slot;
    unsigned char* dst = packed + rec * kPkTileBytes;
    uint32_t* lo = reinterpret_cast<uint32_t*>(dst);
    uint8_t* hi = dst + kTileElems * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const long long mi = __double2ll_rn(v[q] * up);
        const unsigned long long u = (unsigned long long)(mi + (1LL << 39));
        lo[threadIdx.x + 256 * q] = (uint32_t)u;
        hi[threadIdx.x + 256 * q] = (uint8_t)(u >> 32);
    }
    if (threadIdx.x == 0) scales[rec] = ldexp(1.0, e - kPkFrac);
}

cudaError_t launch_pack_pairs_from_panels(const double* rp, int64_t ld_r, const double* cp, int64_t ld_c, int n, int I0,
                                          int pbase, int npairs_local, int k, int l, void* packed, double* scales,
                                          cudaStream_t stream) {
    const int nt = (int)ceil_div(n, kTile);
    if (npairs_local <= 0) return cudaSuccess;
    pack_pairs_from_panels_kernel<<<(unsigned)(2 * npairs_local), 256, 0, stream>>>(
        rp, ld_r, cp, ld_c, n, nt, I0, pbase, k, l, (unsigned char*)packed, scales);
    return cudaGetLastError();
}

// The owner's side of the fused reduce-scatter: out[i] = sum_s slots[s][i] over the G receive
// slots (one per source rank), in rank order (deterministic).
__global__ void __launch_bounds__(256) sum_slots_kernel(const double* __restrict__ slots, int nslots, int64_t count,
                                                        double* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < count; i += (int64_t)gridDim.x * 256) {
        double v = slots[i];
        for (int s = 1; s < nslots; ++s) v += slots[(int64_t)s * count + i];
        out[i] = v;
    }
}

cudaError_t launch_sum_slots(const double* slots, int nslots, int64_t count, double* out, cudaStream_t stream) {
    sum_slots_kernel<<<4 * FGFRFT_SMS, 256, 0, stream>>>(slots, nslots, count, out);
    return cudaGetLastError();
}

size_t packed_bytes_pairs(int64_t npairs, int l) { return (size_t)npairs * (size_t)l * 2 * kPkTileBytes; }

// ---------------------------------------------------------------- MSE + dL/da from [Y; dY]
// loss = ||Y - Xc||^2 / (n b), dL/da = 2 Re<Y - Xc, dY> / (n b)  (G = 2 (Y - Xc) / (n b),
// learn.hpp:85-92 normalisation; dY = dQ/da X, so Re<G, dY> = Re<G, F'^a X>). Fixed-order
// two-pass reduction (deterministic). Optionally copies Y out (the caller's y buffer).
constexpr int kMdBlocks = 4 * FGFRFT_SMS;

__global__ void __launch_bounds__(256) mse_dy_kernel(const double2* __restrict__ y, const double2* __restrict__ dy,
                                                     const double2* __restrict__ xc, int64_t count,
                                                     double2* __restrict__ yout, double* __restrict__ part) {
    __shared__ double red[2][8];
    double s1 = 0.0, s2 = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < count; i += (int64_t)gridDim.x * 256) {
        const double2 v = y[i], d = dy[i], c = xc[i];
        const double rx = v.x - c.x, ry = v.y - c.y;
        s1 = fma(rx, rx, fma(ry, ry, s1));
        s2 = fma(rx, d.x, fma(ry, d.y, s2));
        if (yout) yout[i] = v;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = s1;
        red[1][threadIdx.x >> 5] = s2;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[threadIdx.x][w];
        part[(int64_t)threadIdx.x * kMdBlocks + blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(64) mse_dy_finish_kernel(const double* __restrict__ part, double norm,
                                                           double* __restrict__ loss, double* __restrict__ dlda) {
    __shared__ double red[2][2];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;  // warp 0: loss, warp 1: dot
    double t = 0.0;
    for (int i = lane; i < kMdBlocks; i += 32) t += part[(int64_t)w * kMdBlocks + i];
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[w][0] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        *loss = red[0][0] * norm;
        *dlda = 2.0 * red[1][0] * norm;
    }
}

size_t mse_dy_part_elems() { return 2 * kMdBlocks; }

// Chunked form (host-buffer step: the loss of a column chunk as soon as its Xc has landed): the
// partials of chunk `slot` go to part + slot * mse_dy_part_elems(); launch_mse_dy_finish_n sums
// `nslots` of them in fixed order.
__global__ void __launch_bounds__(64) mse_dy_finish_n_kernel(const double* __restrict__ part, int nslots, double norm,
                                                             double* __restrict__ loss, double* __restrict__ dlda) {
    __shared__ double red[2];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;  // warp 0: loss, warp 1: dot
    double t = 0.0;
    for (int s = 0; s < nslots; ++s)
        for (int i = lane; i < kMdBlocks; i += 32) t += part[((int64_t)s * 2 + w) * kMdBlocks + i];
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[w] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        *loss = red[0] * norm;
        *dlda = 2.0 * red[1] * norm;
    }
}

cudaError_t launch_mse_dy_part(const void* y, const void* dy, const void* xc, int64_t count, void* yout, double* part,
                               int slot, cudaStream_t stream) {
    mse_dy_kernel<<<kMdBlocks, 256, 0, stream>>>((const double2*)y, (const double2*)dy, (const double2*)xc, count,
                                                 (double2*)yout, part + (size_t)slot * 2 * kMdBlocks);
    return cudaGetLastError();
}

cudaError_t launch_mse_dy_finish_n(const double* part, int nslots, double norm, double* loss, double* dlda,
                                   cudaStream_t stream) {
    mse_dy_finish_n_kernel<<<1, 64, 0, stream>>>(part, nslots, norm, loss, dlda);
    return cudaGetLastError();
}

// One CTA per order: fixed-order strided sums (four independent chains per thread) and a fixed tree
// (deterministic run to run).
__global__ void __launch_bounds__(1024) fused_mse_finish_kernel(const double2* __restrict__ part, int64_t per,
                                                                double norm, double* __restrict__ loss,
                                                                double* __restrict__ dlda) {
    __shared__ double red[2][32];
    const double2* p = part + (int64_t)blockIdx.x * per;
    double s1[4] = {0.0, 0.0, 0.0, 0.0}, s2[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t i0 = threadIdx.x; i0 < per; i0 += 4096) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t i = i0 + q * 1024;
            const double2 v = i < per ? p[i] : make_double2(0.0, 0.0);
            s1[q] += v.x;
            s2[q] += v.y;
        }
    }
    double t1 = (s1[0] + s1[1]) + (s1[2] + s1[3]), t2 = (s2[0] + s2[1]) + (s2[2] + s2[3]);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        t1 += __shfl_xor_sync(0xffffffffu, t1, o);
        t2 += __shfl_xor_sync(0xffffffffu, t2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = t1;
        red[1][threadIdx.x >> 5] = t2;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        t1 = red[0][threadIdx.x];
        t2 = red[1][threadIdx.x];
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            t1 += __shfl_xor_sync(0xffffffffu, t1, o);
            t2 += __shfl_xor_sync(0xffffffffu, t2, o);
        }
        if (threadIdx.x == 0) {
            loss[blockIdx.x] = t1 * norm;
            dlda[blockIdx.x] = 2.0 * t2 * norm;
        }
    }
}

cudaError_t launch_fused_mse_finish(const double* part, int64_t per, int n_alpha, double norm, double* loss,
                                    double* dlda, cudaStream_t stream) {
    fused_mse_finish_kernel<<<n_alpha, 1024, 0, stream>>>(reinterpret_cast<const double2*>(part), per, norm, loss, dlda);
    return cudaGetLastError();
}

cudaError_t launch_mse_dy(const void* y, const void* dy, const void* xc, int64_t count, void* yout, double* part,
                          double norm, double* loss, double* dlda, cudaStream_t stream) {
    mse_dy_kernel<<<kMdBlocks, 256, 0, stream>>>((const double2*)y, (const double2*)dy, (const double2*)xc, count,
                                                 (double2*)yout, part);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    mse_dy_finish_kernel<<<1, 64, 0, stream>>>(part, norm, loss, dlda);
    return cudaGetLastError();
}


// ---------------------------------------------------------------- the order window
//
// Node operators of a declared order window [lo, hi] (fgfrft_cache_set_order_window): W'_j =
// sum_{k != 0} c_k(x_j) P_k at the r Chebyshev nodes x_j of the window, exact FP64 (synthesised
// once by the FP64 series kernels), column-major n x n each. Per call, for orders inside the
// window, Q(a) - c_0(a) I = sum_j l_j(a) W'_j and dQ/da - c'_0(a) I = sum_j l_j'(a) W'_j (barycentric
// weights; the c_0 terms come back exactly in the product GEMM's epilogue): r slabs streamed instead
// of the L packed powers. One thread per row over a 64-column chunk, all outputs per staged value;
// row maxima of each output by atomicMax on the ordered bits (the Ozaki slicing reads them).
namespace {
template <int ROWS>
__global__ void __launch_bounds__(256) window_synth_kernel(const double* __restrict__ wops, int r, int n, int64_t nn,
                                                           WindowWeights ww, double* __restrict__ out,
                                                           int64_t ostride, unsigned long long* __restrict__ rowmax,
                                                           int64_t mp, int row0, int row1) {
    const int i = row0 + blockIdx.x * 256 + threadIdx.x;
    const int j0 = blockIdx.y * 64, j1 = min(j0 + 64, n);
    if (i >= row1) return;
    double mx[ROWS];
#pragma unroll
    for (int x = 0; x < ROWS; ++x) mx[x] = 0.0;
    // two columns per pass, 16 node operators per batch of loads: 32 independent 8-byte loads in
    // flight per thread before the first FMA (the first form, one load chain per column, ran at 0.60
    // of the DRAM peak on long-scoreboard stalls)
    for (int j = j0; j < j1; j += 2) {
        const bool two = j + 1 < j1;
        const double* p0 = wops + (int64_t)j * n + i;
        const double* p1 = p0 + n;
        double a0[ROWS], a1[ROWS];
#pragma unroll
        for (int x = 0; x < ROWS; ++x) a0[x] = a1[x] = 0.0;
        for (int t0 = 0; t0 < r; t0 += 16) {
            double v0[16], v1[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int t = t0 + u;
                v0[u] = t < r ? __ldcs(p0 + (int64_t)t * nn) : 0.0;
                v1[u] = (t < r && two) ? __ldcs(p1 + (int64_t)t * nn) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                if (t0 + u >= r) break;
#pragma unroll
                for (int x = 0; x < ROWS; ++x) {
                    a0[x] = fma(ww.w[x][t0 + u], v0[u], a0[x]);
                    a1[x] = fma(ww.w[x][t0 + u], v1[u], a1[x]);
                }
            }
        }
#pragma unroll
        for (int x = 0; x < ROWS; ++x) {
            __stcs(out + x * ostride + (int64_t)j * n + i, a0[x]);
            mx[x] = fmax(mx[x], fabs(a0[x]));
            if (two) {
                __stcs(out + x * ostride + (int64_t)(j + 1) * n + i, a1[x]);
                mx[x] = fmax(mx[x], fabs(a1[x]));
            }
        }
    }
#pragma unroll
    for (int x = 0; x < ROWS; ++x)
        if (mx[x] > 0.0) atomicMax(rowmax + x * mp + i, (unsigned long long)__double_as_longlong(mx[x]));
}
}  // namespace

cudaError_t launch_window_synth(const double* wops, int r, int n, const WindowWeights& ww, int rows, double* out,
                                int64_t ostride, unsigned long long* rowmax, int64_t mp, cudaStream_t stream,
                                int row0, int row1) {
    if (r < 1 || r > kWindowMaxNodes) return cudaErrorInvalidValue;
    if (row1 < 0 || row1 > n) row1 = n;
    if (row1 <= row0) return cudaSuccess;
    const dim3 grid((unsigned)ceil_div(row1 - row0, 256), (unsigned)ceil_div(n, 64));
    const int64_t nn = (int64_t)n * n;
    switch (rows) {
        case 1: window_synth_kernel<1><<<grid, 256, 0, stream>>>(wops, r, n, nn, ww, out, ostride, rowmax, mp, row0, row1); break;
        case 2: window_synth_kernel<2><<<grid, 256, 0, stream>>>(wops, r, n, nn, ww, out, ostride, rowmax, mp, row0, row1); break;
        case 4: window_synth_kernel<4><<<grid, 256, 0, stream>>>(wops, r, n, nn, ww, out, ostride, rowmax, mp, row0, row1); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace fgb
