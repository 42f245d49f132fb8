// ozgemm.cu -- FP64-accurate real GEMM on the INT8 tensor cores (Ozaki scheme, tcgen05).
//
// sm_100a has no FP64 tcgen05 kind: the FP64 tensor path is warp-level DMMA at ~37 TFLOP/s,
// while tcgen05.mma kind::i8 runs ~4.5 POPS with int32 accumulators in TMEM. An FP64 product
// C = A B^T (A: M x K, B: N x K) is computed exactly-in-int8 by fixed-point slicing:
//   every row r of A is scaled by 2^-(e_r+1) (max |a_r.| < 2^e_r) and cut into S balanced
//   base-254 digits,  a_rk = 2^(e_r+1) * sum_{t=1..S} A_t[r,k] 254^-t,  |A_t| <= 127  (rint
//   digits; remainders exact to 2^-53); B likewise per row. Then
//   C = 2^(e_r + e_n + 2) * sum_{t+u <= S+1} 254^-(t+u) (A_t B_u^T), where every int8 GEMM is
//   exact in int32 (K * 127^2 * S < 2^31 for K <= 16384). Dropped terms and truncated digits
//   bound the error by ~ sqrt(K) 254^-S of |row max| |col max|: S = 6 (21 digit products)
//   gives 3e-13 relative on the BASELINE configs (DMMA: ~1e-15; the parity bar is 1e-10),
//   S = 7 (28 products) ~1e-15.
//
// Kernel layout (one 128 x 64 output tile per CTA, 256 threads):
//   * operands are pre-sliced by oz_slice_kernel into the tcgen05 canonical no-swizzle K-major
//     layout, blocked so that one (tile, 64-byte K block) of ALL S slices is ONE contiguous
//     chunk: a stage is two 1-D bulk copies (UBLKCP) onto an mbarrier;
//   * S int32 accumulators, one per digit weight d = t + u (2..S+1), live side by side in TMEM
//     (S x 64 columns <= 512). For a fixed A digit t the B digits u = 1..S+1-t are stacked
//     along N in shared memory, so ONE tcgen05.mma (N up to 256) covers a contiguous run of
//     accumulators: 9 MMAs per 32-byte K step for S = 6 (21 digit products);
//   * a 3-4 stage ring of 64- / 32-byte K blocks; warp 0 / lane 0 issues the bulk copies, warp 1 / lane 0
//     the MMAs (tcgen05.commit frees a stage), then all 8 warps drain TMEM (tcgen05.ld 32x32b,
//     lane = output row, 32 columns per warp) and combine the S accumulators in FP64 (Horner
//     in base 254 over exact int64 folds) into the output.
#include "oz.cuh"
#include "tc.cuh"

#include <cstdlib>

namespace fgb {

constexpr int kOzBM = 128;  // rows of the A tile (TMEM lanes)
constexpr int kOzBN = 64;   // rows of the B tile (N of one digit product)

// Digit base 254: with |v| < 1/2, rint(254 v) is in [-127, 127] and the remainder in [-1/2, 1/2],
// so every digit fits int8 and carries log2(254) = 7.99 bits (base 256 would need 128).
constexpr double kOzBase = 254.0;
constexpr long long kOzBaseI = 254;
constexpr double kOzMagic = 6755399441055744.0;  // 1.5 * 2^52: x + magic rounds x (|x| < 2^51) to an integer
constexpr int kOzZDigits = 7;  // digits of Z written by the CM 2 epilogue (bounded by column norms: +1 digit)
constexpr double kOzScale = 4.0 / (254.0 * 254.0 * 254.0 * 254.0);  // 2^2 (two half scalings) x 254^-4
__host__ __device__ constexpr double oz_pow254(int k) { return k == 0 ? 1.0 : 254.0 * oz_pow254(k - 1); }

// Stage geometry per digit count: 6 digits -> 64-byte K blocks (two MMA K steps, 18 MMAs per
// stage) in a 3-stage ring; 7-8 digits -> 32-byte K blocks in a 5- / 4-stage ring (<= 219 KB smem).
template <int S, int BN = kOzBN, bool P = false> struct OzCfg {
    static constexpr int bk = S <= 6 ? 64 : 32;        // bytes (= int8 elements) of K per stage
    static constexpr int stages = S <= 6 ? 3 : (S == 7 ? 5 : 4);
    static constexpr int sbo = bk / 16 * 128;          // bytes between 8-row groups of a slice block
    static constexpr int a_stage = S * kOzBM * bk;
    static constexpr int b_stage = S * BN * bk;
    static constexpr int stage = a_stage + b_stage;
    // + barriers / scratch + CM 2 exchange (+ the narrow form's pair-mode row maxima, [2][32][32])
    static constexpr int smem = stages * stage + 1024 + 2048 + (P ? 16384 : 0);
};


__device__ __forceinline__ double pow2(int e) {  // exact 2^e for -1022 <= e <= 1023
    return __longlong_as_double((long long)(e + 1023) << 52);
}

// ---------------------------------------------------------------- operand views and slicing (OzView: oz.cuh)

__device__ __forceinline__ double oz_load(const OzView& v, int row, int k) {
    if (v.tiled == 5) {  // complex product operand (see OzView)
        const int bt = row / v.rp, r = row - bt * v.rp;
        if (r >= v.rv || k >= v.kv) return 0.0;
        const int kc = k >> 1, e = k & 1;
        const int rc = v.ra ? r >> 1 : r, c = v.ra ? r & 1 : 0;
        const double2 z = reinterpret_cast<const double2*>(v.src)[bt * v.sbatch + (int64_t)rc * v.rs + (int64_t)kc * v.ks];
        const double zr = z.x, zi = v.ka ? -z.y : z.y;
        if (!v.ra) return e ? -zi : zr;
        return c == 0 ? (e ? zi : zr) : (e ? -zr : zi);
    }
    if (v.tiled == 6) {  // element rows of the stacked cache: row e = i + j n, K term kk (see OzView)
        if (row >= v.rv || k >= v.kv || k >= 2 * v.l) return 0.0;
        const int n = v.tp2, i = row % n, j = row / n;
        const bool tr = k >= v.l;
        const int slab = tr ? k - v.l : k;
        const int a = tr ? j : i, b = tr ? i : j;
        return v.src[slab * v.sbatch + tile_base(a >> 5, b >> 5, v.nt) + swz(a & 31, b & 31)];
    }
    if (v.tiled == 7) {  // element-pair rows of the digit cache (see OzView)
        if (row >= v.rv || k >= v.kp) return 0.0;
        const int mt = row >> 7, p = mt >> 3;
        const int t = 128 * (mt & 7) + (row & 127), kh = v.kp >> 1;
        const bool mirror = k >= kh;
        const int kk = mirror ? k - kh : k;
        if (kk >= v.l) return 0.0;
        int I, J;
        pair_of_imajor(p, v.nt, I, J);
        const int i = t & 31, j = t >> 5;
        const int gr = mirror ? J * 32 + j : I * 32 + i, gc = mirror ? I * 32 + i : J * 32 + j;
        if (gr >= v.tp2 || gc >= v.tp2) return 0.0;
        return v.src[(int64_t)kk * v.sbatch + tile_base(gr >> 5, gc >> 5, v.nt) + swz(gr & 31, gc & 31)];
    }
    if (v.tiled == 3) {  // rv = n (signal rows), rows beyond n * tp2 are padding
        const int i = row / v.tp2, kk = row - i * v.tp2;
        if (i >= v.rv || kk >= 2 * v.l || k >= v.kv) return 0.0;
        const bool tr = kk >= v.l;
        const int slab = tr ? kk - v.l : kk;
        const int a = tr ? k : i, b = tr ? i : k;
        return v.src[slab * v.sbatch + tile_base(a >> 5, b >> 5, v.nt) + swz(a & 31, b & 31)];
    }
    const int bt = row / v.rp, r = row - bt * v.rp;
    if (r >= v.rv || k >= v.kv) return 0.0;
    if (v.tiled == 8) {
        const int x = r >> 1, kh = v.kp >> 1;
        const bool hi = k >= kh;
        const int kk = hi ? k - kh : k;
        if (kk >= v.l) return 0.0;
        const bool neg = hi != (bool)(r & 1);
        return v.src[(int64_t)x * v.rs + v.l + (neg ? -(kk + 1) : kk + 1)];
    }
    if (v.tiled == 4) {
        const int kk = k;
        if (kk >= 2 * v.l) return 0.0;
        const int q = kk < v.l ? v.l + 1 + kk : 2 * v.l - 1 - kk;
        return v.src[(int64_t)r * v.rs + q];
    }
    if (v.tiled) {
        const int i = v.tiled == 1 ? r : k, j = v.tiled == 1 ? k : r;
        return v.src[bt * v.sbatch + tile_base(i >> 5, j >> 5, v.nt) + swz(i & 31, j & 31)];
    }
    return v.src[bt * v.sbatch + (int64_t)(r >> v.ra) * v.rs + (r & v.ra) + (int64_t)(k >> v.ka) * v.ks + (k & v.ka)];
}

// 64 x 64 tile of the operand -> shared [64][65], coalesced along the contiguous direction.
__device__ __forceinline__ void oz_tile_load(const OzView& v, int row0, int k0, double (*t)[65]) {
    for (int idx = threadIdx.x; idx < 64 * 64; idx += blockDim.x) {
        const int a = idx & 63, b = idx >> 6;
        const int r = v.rfast ? a : b, k = v.rfast ? b : a;
        t[r][k] = oz_load(v, row0 + r, k0 + k);
    }
}

// Row-max slot of sliced row `row` (= bt * rp + r): bt * rmb + r when the view sets rmb.
__device__ __forceinline__ int64_t oz_rm_index(const OzView& v, int row) {
    if (!v.rmb) return row;
    const int bt = row / v.rp;
    return (int64_t)bt * v.rmb + (row - bt * v.rp);
}

// Pass 1: per-row max |a| (as ordered bits of a non-negative double) via atomicMax.
__global__ void __launch_bounds__(256) oz_rowmax_kernel(OzView v, unsigned long long* rowmax) {
    __shared__ double t[64][65];
    const int row0 = blockIdx.x * 64, k0 = blockIdx.y * 64;
    oz_tile_load(v, row0, k0, t);
    __syncthreads();
    const int r = threadIdx.x >> 2, q = threadIdx.x & 3;  // 4 threads per row
    double m = 0.0;
#pragma unroll 4
    for (int k = q; k < 64; k += 4) m = fmax(m, fabs(t[r][k]));
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 1));
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 2));
    if (q == 0 && m > 0.0) atomicMax(rowmax + row0 + r, (unsigned long long)__double_as_longlong(m));
}

// Pass 2: digits. Output chunk for (row tile rt of TR rows, 32-byte K block kb):
//   dst + ((rt * KB + kb) * S + t) * TR * 32  +  g * 256 + c * 128 + r8 * 16 + (k & 15)
// with g = (row % TR) / 8, r8 = row % 8, c = (k % 32) / 16 -- the canonical no-swizzle K-major
// layout with SBO = 256 B (8-row groups) and LBO = 128 B (16-byte K chunks). All S slices of
// one (row tile, K block) are contiguous: one bulk copy per operand and pipeline stage.
template <int S>
__global__ void __launch_bounds__(256) oz_slice_kernel(OzView v, const unsigned long long* rowmax, int tr,
                                                       int8_t* __restrict__ dst, int* __restrict__ exps) {
    __shared__ double t[64][65];
    const int row0 = blockIdx.x * 64, k0 = blockIdx.y * 64;
    oz_tile_load(v, row0, k0, t);
    __syncthreads();
    const int u = threadIdx.x;  // (g_local, c, r8): one 16-byte digit run per thread and slice
    const int gl = u >> 5, c = (u >> 3) & 3, r8 = u & 7;
    const int rl = gl * 8 + r8, row = row0 + rl;
    const double mx = __longlong_as_double((long long)rowmax[oz_rm_index(v, row)]);
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
    if (blockIdx.y == 0 && c == 0) exps[row] = e;
    const double sc = mx > 0.0 ? pow2(-e - 1) : 0.0;  // |a| * sc < 1/2
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = t[rl][c * 16 + i] * sc;
    constexpr int kBK = OzCfg<S>::bk;
    const int kb_count = v.kp / kBK;
    const int rt = row / tr, rr = row - rt * tr;
    const int kb = (blockIdx.y * 64 + c * 16) / kBK, cl = c & (kBK / 16 - 1);
    int8_t* base = dst + ((int64_t)rt * kb_count + kb) * S * tr * kBK + (rr >> 3) * OzCfg<S>::sbo + cl * 128 + r8 * 16;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t packed = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double y = x[q * 4 + i] * kOzBase;  // |y| <= 127
                const double t = y + kOzMagic;            // rint(y) in the low word
                x[q * 4 + i] = y - (t - kOzMagic);        // exact, |.| <= 1/2
                packed |= ((uint32_t)__double2loint(t) & 0xFFu) << (8 * i);
            }
            w[q] = packed;
        }
        *reinterpret_cast<uint4*>(base + (int64_t)s * tr * kBK) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// Direct forms for plain strided views whose rows are the contiguous direction (rfast: Q, G and
// the products' operands): one thread per row, 64 K values per block, loads coalesced across
// the warp's consecutive rows, no shared-memory staging (the tile forms above were issue-bound).
__device__ __forceinline__ const double* oz_row_ptr(const OzView& v, int row, bool* valid) {
    const int bt = row / v.rp, rr = row - bt * v.rp;
    *valid = rr < v.rv;
    return v.src + (int64_t)bt * v.sbatch + (int64_t)(rr >> v.ra) * v.rs + (rr & v.ra);
}

__global__ void __launch_bounds__(64) oz_rowmax_direct_kernel(OzView v, unsigned long long* rowmax) {
    const int row = blockIdx.x * 64 + threadIdx.x, k0 = blockIdx.y * 64;
    bool ok;
    const double* p = oz_row_ptr(v, row, &ok);
    if (!ok) return;
    const int kn = min(64, v.kv - k0);
    double m = 0.0;
#pragma unroll 8
    for (int i = 0; i < kn; ++i) {
        const int k = k0 + i;
        m = fmax(m, fabs(p[(int64_t)(k >> v.ka) * v.ks + (k & v.ka)]));
    }
    if (m > 0.0) atomicMax(rowmax + row, (unsigned long long)__double_as_longlong(m));
}

// S digit slices of one 16-byte run (K = k0 .. k0 + 15 of row (rt, rr)) from its scaled values.
template <int S>
__device__ __forceinline__ void oz_write_digits(double (&x)[16], int kp, int k0, int tr, int rt, int rr,
                                                int8_t* __restrict__ dst) {
    constexpr int kBK = OzCfg<S>::bk;
    const int kb_count = kp / kBK;
    const int kb = k0 / kBK, cl = (k0 >> 4) & (kBK / 16 - 1);
    int8_t* base = dst + ((int64_t)rt * kb_count + kb) * S * tr * kBK + (rr >> 3) * OzCfg<S>::sbo + cl * 128 + (rr & 7) * 16;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t packed = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double y = x[q * 4 + i] * kOzBase;
                const double t = y + kOzMagic;
                x[q * 4 + i] = y - (t - kOzMagic);
                packed |= ((uint32_t)__double2loint(t) & 0xFFu) << (8 * i);
            }
            w[q] = packed;
        }
        *reinterpret_cast<uint4*>(base + (int64_t)s * tr * kBK) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// One 16-byte digit run of a plain strided view -> S digit slices.
template <int S>
__device__ __forceinline__ void oz_digit_run(const OzView& v, const double* p, bool ok, double sc, int k0, int tr,
                                             int rt, int rr, int8_t* __restrict__ dst) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int k = k0 + i;
        x[i] = (ok && k < v.kv) ? p[(int64_t)(k >> v.ka) * v.ks + (k & v.ka)] * sc : 0.0;
    }
    oz_write_digits<S>(x, v.kp, k0, tr, rt, rr, dst);
}

template <int S>
__global__ void __launch_bounds__(64) oz_slice_direct_kernel(OzView v, const unsigned long long* rowmax, int tr,
                                                             int8_t* __restrict__ dst, int* __restrict__ exps) {
    const int row = blockIdx.x * 64 + threadIdx.x, k0 = blockIdx.y * 64;
    bool ok;
    const double* p = oz_row_ptr(v, row, &ok);
    const double mx = __longlong_as_double((long long)rowmax[oz_rm_index(v, row)]);
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
    if (blockIdx.y == 0) exps[row] = e;
    const double sc = mx > 0.0 ? pow2(-e - 1) : 0.0;  // |a| * sc < 1/2
    const int rt = row / tr, rr = row - rt * tr;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) oz_digit_run<S>(v, p, ok, sc, k0 + c * 16, tr, rt, rr, dst);  // K = k0 + 16c ..
}

// Row max and digits in ONE kernel for tall row-contiguous views (the node operators W_j: 19n
// rows): a CTA owns 32 rows and all of K, its 8 warps take interleaved 64-wide K blocks (lanes =
// consecutive rows, coalesced), reduce the row max through shared memory, then slice the same
// blocks -- the second read of the CTA's 32 rows is an L2 hit, so W crosses HBM once instead of
// twice, and there is no rowmax memset / atomic pass.
template <int S>
__global__ void __launch_bounds__(256) oz_rowslice_direct_kernel(OzView v, int tr, int8_t* __restrict__ dst,
                                                                 int* __restrict__ exps) {
    __shared__ double wmax[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int row = blockIdx.x * 32 + lane, kblocks = v.kp / 64;
    bool ok;
    const double* p = oz_row_ptr(v, row, &ok);
    double m = 0.0;
    if (ok)
        for (int kb = w; kb < kblocks; kb += 8) {
            const int k0 = kb * 64, kn = min(64, v.kv - k0);
#pragma unroll 8
            for (int i = 0; i < kn; ++i) {
                const int k = k0 + i;
                m = fmax(m, fabs(p[(int64_t)(k >> v.ka) * v.ks + (k & v.ka)]));
            }
        }
    wmax[w][lane] = m;
    __syncthreads();
    double mx = wmax[0][lane];
#pragma unroll
    for (int q = 1; q < 8; ++q) mx = fmax(mx, wmax[q][lane]);
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
    if (w == 0) exps[row] = e;
    const double sc = mx > 0.0 ? pow2(-e - 1) : 0.0;  // |a| * sc < 1/2
    const int rt = row / tr, rr = row - rt * tr;
    // slice in the reverse order of the max pass: the most recently read K blocks are the likeliest
    // L2 hits
    for (int kb = w + (kblocks - 1 - w) / 8 * 8; kb >= 0; kb -= 8)
#pragma unroll 1
        for (int c = 3; c >= 0; --c) oz_digit_run<S>(v, p, ok, sc, kb * 64 + c * 16, tr, rt, rr, dst);
}

// Complex signal columns as B-operand row pairs (rows 2j, 2j + 1 = Re, Im of column j, K = the
// signal index, interleaved (re, im) in memory): a 64-thread block per column, thread = 16-wide K
// runs; the row max of both rows by shuffles + shared memory, then the digits from a second read
// of the (L1/L2-resident) column. One kernel, no memset / atomics.
template <int S>
__global__ void __launch_bounds__(64) oz_rowslice_pairs_kernel(OzView v, int tr, int8_t* __restrict__ dst,
                                                               int* __restrict__ exps) {
    __shared__ double wm[2][2];
    const int t = threadIdx.x, lane = t & 31, j = blockIdx.x;
    const int r0 = 2 * j;
    const bool ok = r0 < v.rv;  // rv even (2 x columns)
    const double2* col = reinterpret_cast<const double2*>(v.src + (int64_t)j * v.rs);
    const int runs = v.kp / 16;
    double m0 = 0.0, m1 = 0.0;
    if (ok)
        for (int q = t; q < runs; q += 64)
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int k = q * 16 + i;
                if (k < v.kv) {
                    const double2 z = col[k];
                    m0 = fmax(m0, fabs(z.x));
                    m1 = fmax(m1, fabs(z.y));
                }
            }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        m0 = fmax(m0, __shfl_xor_sync(0xffffffffu, m0, o));
        m1 = fmax(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    }
    if (lane == 0) {
        wm[t >> 5][0] = m0;
        wm[t >> 5][1] = m1;
    }
    __syncthreads();
    m0 = fmax(wm[0][0], wm[1][0]);
    m1 = fmax(wm[0][1], wm[1][1]);
    int e0 = 0, e1 = 0;
    if (m0 > 0.0) frexp(m0, &e0);
    if (m1 > 0.0) frexp(m1, &e1);
    if (t == 0) {
        exps[r0] = e0;
        exps[r0 + 1] = e1;
    }
    const double s0 = m0 > 0.0 ? pow2(-e0 - 1) : 0.0, s1 = m1 > 0.0 ? pow2(-e1 - 1) : 0.0;
    const int rt0 = r0 / tr, rr0 = r0 - rt0 * tr, rt1 = (r0 + 1) / tr, rr1 = r0 + 1 - rt1 * tr;
    for (int q = t; q < runs; q += 64) {
        double x0[16], x1[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int k = q * 16 + i;
            const double2 z = (ok && k < v.kv) ? col[k] : make_double2(0.0, 0.0);
            x0[i] = z.x * s0;
            x1[i] = z.y * s1;
        }
        oz_write_digits<S>(x0, v.kp, q * 16, tr, rt0, rr0, dst);
        oz_write_digits<S>(x1, v.kp, q * 16, tr, rt1, rr1, dst);
    }
}

// ---------------------------------------------------------------- the GEMM



constexpr int kOzEpiWarps = 16;                       // 4 TMEM lane groups x 4 column quarters
constexpr int kOzEpiQ = kOzEpiWarps / 4;              // column groups
constexpr int kOzEC = kOzBN / kOzEpiQ;                // columns per epilogue thread (16)
constexpr int kOzThreads = 32 * (2 + kOzEpiWarps);    // producer warp, MMA warp, epilogue warps

// Persistent, clusters of CL CTAs along N (CL = 2 by default): cluster c owns work units u = c, c + clusters, ...
// (unit = one A row tile x CL adjacent N tiles; CTA rank r computes N tile r of the unit).
// Every A stage is fetched ONCE per cluster: CTA r bulk-copies slice r/CL of it with
// .multicast::cluster into all CL CTAs; each CTA's MMA commit arrives on every CTA's `empty`
// barrier (count CL), so a stage is refilled only after the whole cluster consumed it.
// Warp 0 streams K blocks of consecutive units through the stage ring without a break; warp 1
// issues the MMAs of a tile once the epilogue has drained the previous accumulators
// (tmem_empty); warps 2..9 drain TMEM, fold the S int32 accumulators into two exact int64
// partial sums, release TMEM and only then convert, scale and store -- so the FP64 epilogue
// overlaps the next tile's MMAs.
// BN = 32 (CM 0 only): the skinny node-operator form -- B tiles of 32 rows (r <= 32 live output
// columns), S x 32 TMEM columns per accumulator set, so two sets fit and the MMAs of unit u + 1
// run while the epilogue drains unit u (tfull / tempty per buffer).
// P: the element-pair node-operator mode (OzOut::pair_nt, narrow form only) -- a separate
// instantiation so its registers do not burden the default forms.
template <int S, int CM, int CL, int BN = kOzBN, bool P = false>
__global__ void __launch_bounds__(kOzThreads, 1)
ozgemm_kernel(const int8_t* __restrict__ a, const int* __restrict__ ea, const int8_t* __restrict__ b,
              const int* __restrict__ eb, int kblocks, int mtiles, int ntiles, OzOut out) {
    static_assert(BN == kOzBN || (BN == 32 && CM == 0), "narrow tiles: node operators only");
    static_assert(!P || (BN == 32 && CM == 0 && CL == 1), "pair mode: the narrow form");
    using Cfg = OzCfg<S, BN, P>;
    constexpr int NB = BN == kOzBN ? 1 : 2;        // TMEM accumulator buffers
    constexpr uint32_t kBufCols = BN == kOzBN ? 0 : 256;
    constexpr int kOzStages = Cfg::stages;
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* sa = smem;
    unsigned char* sb = smem + kOzStages * Cfg::a_stage;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOzStages * Cfg::stage);
    uint64_t* empty = full + kOzStages;
    uint64_t* tfull = empty + kOzStages;  // [NB]
    uint64_t* tempty = tfull + 2;         // [NB]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    double* xchg = reinterpret_cast<double*>(smem + kOzStages * Cfg::stage + 1024);  // CM 2: 2 x [2][64]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = CL > 1 ? (int)cluster_rank() : 0;
    const int cid = blockIdx.x / CL, nclusters = gridDim.x / CL;
    const int ngroups = ntiles / CL, units = mtiles * ngroups;
    constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1);
    constexpr int kAPart = Cfg::a_stage / CL;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kOzStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, CL);
        }
        for (int q = 0; q < NB; ++q) {
            mbar_init(tfull + q, 1);
            mbar_init(tempty + q, kOzEpiWarps);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    if (CL > 1) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // unit schedule: strided over the clusters. Row-max node operators (out.rmax): the host sizes
    // the grid as a multiple of the row blocks per column (rn / 128), so every unit of a CTA lies in
    // the same row block and the row max stays in registers until one flush at the end
    // pair mode (out.pair_nt): a CTA takes the 8 M tiles of one tile pair in a row (row maxima of
    // the pair's rows stay in registers across them)
    constexpr bool pairs = P;
    const bool chunk = CM == 0 && CL == 1 && out.rmax != nullptr && out.nv <= 32 && !pairs;  // (the skinny epilogue)
    const int upp = 8 * ngroups;  // pair mode: units of one tile pair (8 M tiles x the N tiles)
    // fused MSE (CM 1, out.lpart): units 2 pu (Y tile) and 2 pu + 1 (its dY tile) back to back per CTA
    const bool fmse = CM == 1 && out.lpart != nullptr;
    const int mhalf = mtiles >> 1;
    const int ub = pairs ? cid * upp : (fmse ? 2 * cid : cid), ue = units, us = nclusters;
    auto next_u = [&](int u) {
        if (fmse) return (u & 1) ? u - 1 + 2 * us : u + 1;
        return pairs ? ((u % upp) == upp - 1 ? u + upp * us - (upp - 1) : u + 1) : u + us;
    };
    // N bands (CM 1, out.nband > 1): unit q -> band q / (M tiles x gw), then M-major inside the band
    const int gw = (CM == 1 && out.nband > 1) ? ngroups / out.nband : ngroups;
    const int bandu = (fmse ? mhalf : mtiles) * gw;
    auto unit_mt = [&](int u) {
        const int q = fmse ? (u >> 1) : u;
        return (q % bandu) / gw + ((fmse && (u & 1)) ? mhalf : 0);
    };
    auto unit_nt = [&](int u) {
        const int q = fmse ? (u >> 1) : u;
        return ((q / bandu) * gw + q % gw) * CL + rank;
    };

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t keep = policy_evict_last();  // B (the small operand) is reread by every A tile
            int it = 0;  // global K-block counter across units
            for (int u = ub; u < ue; u = next_u(u)) {
                const int mt = unit_mt(u), nt = unit_nt(u);
                const unsigned char* ga = reinterpret_cast<const unsigned char*>(a) + (int64_t)mt * kblocks * Cfg::a_stage;
                const unsigned char* gb = reinterpret_cast<const unsigned char*>(b) + (int64_t)nt * kblocks * Cfg::b_stage;
                for (int kb = 0; kb < kblocks; ++kb, ++it) {
                    const int s = it % kOzStages;
                    if (it >= kOzStages) mbar_wait(empty + s, ((it / kOzStages) - 1) & 1);
                    mbar_arrive_expect_tx(full + s, Cfg::stage);
                    if (CL > 1)
                        bulk_g2s_mc(sa + s * Cfg::a_stage + rank * kAPart, ga + (int64_t)kb * Cfg::a_stage + rank * kAPart,
                                    kAPart, full + s, kMask);
                    else
                        bulk_g2s(sa + s * Cfg::a_stage, ga + (int64_t)kb * Cfg::a_stage, Cfg::a_stage, full + s);
                    bulk_g2s_hint(sb + s * Cfg::b_stage, gb + (int64_t)kb * Cfg::b_stage, Cfg::b_stage, full + s, keep);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int it = 0, tcount = 0;
            for (int u = ub; u < ue; u = next_u(u), ++tcount) {
                const int buf = tcount % NB;
                if (tcount >= NB) mbar_wait(tempty + buf, ((tcount / NB) - 1) & 1);  // epilogue drained it
                tc_fence_after();
                const uint32_t acc = tmem + (uint32_t)buf * kBufCols;
                for (int kb = 0; kb < kblocks; ++kb, ++it) {
                    const int s = it % kOzStages;
                    mbar_wait(full + s, (it / kOzStages) & 1);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sa + s * Cfg::a_stage), b0 = smem_u32(sb + s * Cfg::b_stage);
#pragma unroll
                    for (int j = 0; j < Cfg::bk / 32; ++j) {
#pragma unroll
                        for (int t = 1; t <= S; ++t) {
                            const uint64_t ad = umma_desc(a0 + (t - 1) * kOzBM * Cfg::bk + j * 256, 128, Cfg::sbo);
#pragma unroll
                            for (int u0 = 1; u0 <= S + 1 - t; u0 += 4) {
                                const int cnt = (S + 1 - t - u0 + 1) < 4 ? (S + 1 - t - u0 + 1) : 4;
                                const uint64_t bd = umma_desc(b0 + (u0 - 1) * BN * Cfg::bk + j * 256, 128, Cfg::sbo);
                                const uint32_t col = acc + (uint32_t)((t + u0 - 2) * BN);
                                mma_i8(col, ad, bd, idesc_i8(kOzBM, cnt * BN), (kb > 0 || j > 0 || t > 1) ? 1u : 0u);
                            }
                        }
                    }
                    if (CL > 1) mma_commit_mc(empty + s, kMask); else mma_commit(empty + s);
                }
                mma_commit(tfull + buf);
            }
        }
    } else {
        // epilogue warps 2..17: lane group (warp % 4) = TMEM lanes / output rows, column quarter
        const int ew = warp - 2, lg = warp & 3, h = ew >> 2;
        const int lrow = lg * 32 + lane;
        const uint32_t lane_addr = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(h * kOzEC);
        int tcount = 0;
        double gacc[3] = {0.0, 0.0, 0.0};
        double ls1 = 0.0, ls2 = 0.0;       // CM 1 fused MSE: sum |Y - Xc|^2, sum Re conj(Y - Xc) dY  // CM 2: <X, Z_kk>, <Xc, Z_kk>, <Z_L, Z_kk> over this thread's tiles
        double lacc[kOzEC];                // CM 3: sum (Y - Xc)^2 per order column
        if (CM == 3) {
#pragma unroll
            for (int c = 0; c < kOzEC; ++c) lacc[c] = 0.0;
        }
        // pair mode: the column scales 2^e_n and the diagonal terms in shared memory (the CM 2
        // exchange region), the next unit's row exponent prefetched, the pair's (I, J) per pair
        int ea_nx = 0, pI = 0, pJ = 0;
        // narrow pair mode: the pair's row maxima reduced in shared memory ([mirror][node][row of the
        // tile]) and flushed to global once per pair
        unsigned long long* psm = reinterpret_cast<unsigned long long*>(smem + kOzStages * Cfg::stage + 1024 + 2048);
        if (CM == 0 && BN != kOzBN) {  // narrow forms: column scales / diagonal in shared memory
            const int ndg = pairs ? out.nv / 2 : out.nv;
            for (int t = threadIdx.x - 64; t < kOzBN + 32; t += 32 * kOzEpiWarps)
                xchg[t] = t < kOzBN ? (t < ngroups * BN ? pow2(eb[t]) : 0.0)
                                    : (out.dg && t - kOzBN < ndg ? out.dg[t - kOzBN] : 0.0);
            if (pairs)
                for (int t = threadIdx.x - 64; t < 2048; t += 32 * kOzEpiWarps) psm[t] = 0ull;
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kOzEpiWarps) : "memory");
            if (ub < ue) ea_nx = ea[unit_mt(ub) * kOzBM + lrow];
        }
        auto pair_flush = [&](int I, int J) {  // every epilogue thread, at a pair boundary
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kOzEpiWarps) : "memory");
            for (int t = threadIdx.x - 64; t < 2048; t += 32 * kOzEpiWarps) {
                const unsigned long long v = psm[t];
                if (!v) continue;
                psm[t] = 0ull;
                const int side = t >> 10, x = (t >> 5) & 31, idx = t & 31;
                const int row = (side ? J : I) * 32 + idx;
                if (row < out.pair_n) atomicMax(out.rmax + (int64_t)x * out.rnp + row, v);
            }
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kOzEpiWarps) : "memory");
        };
        double rmx[8];  // chunk mode: running row max of this thread's 8 columns over the row block
        int rib = -1;
        auto flush_rmax = [&](int live) {
            if (rib < 0) return;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < live && rmx[q] > 0.0)
                    atomicMax(out.rmax + (int64_t)(h * ((out.nv + 3) >> 2) + q) * out.rnp + rib * kOzBM + lrow,
                              (unsigned long long)__double_as_longlong(rmx[q]));
        };
        for (int u = ub; u < ue; u = next_u(u), ++tcount) {
            const int mt = unit_mt(u), nt = unit_nt(u);
            const int buf = tcount % NB;
            if (CM == 0 && pairs && BN != kOzBN && (u % upp) == 0) {
                if (tcount > 0 && out.rmax) pair_flush(pI, pJ);
                pair_of_imajor(mt >> 3, out.pair_nt, pI, pJ);
            }
            mbar_wait(tfull + buf, (tcount / NB) & 1);
            tc_fence_after();
            constexpr double lo_w = 1.0 / oz_pow254(S - 3);  // weight of the low fold
            if (BN != kOzBN || (CM == 0 && out.npeers == 0 && out.nv - nt * kOzBN <= 32 && !pairs)) {
                // Skinny output (the node operators: r <= 32 of the 64 tile columns are real): the w
                // live columns are split evenly over the 4 column warps (warp h owns cw = ceil(w / 4)
                // columns from h cw), so only live columns are drained and folded and the per-unit
                // epilogue (the critical path of this HBM-streaming GEMM) is ceil(w / 4) columns deep.
                // All S accumulators are read before TMEM is released, so the next unit's MMAs
                // overlap the whole fold + store instead of waiting for it.
                const int wl = min(out.nv - nt * BN, 32), cw = (wl + 3) >> 2;
                const int c0 = h * cw, live = min(cw, wl - c0);
                double val8[8];
                if (live > 0) {
                    int32_t v[S][8];
#pragma unroll
                    for (int d = 0; d < S; ++d)
                        tmem_ld8(tmem + buf * kBufCols + ((uint32_t)(lg * 32) << 16) + (uint32_t)(d * BN + c0), v[d]);
                    tmem_wait_ld();
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (q >= live) break;
                        long long hi = v[0][q], lo = v[3][q];
                        hi = hi * kOzBaseI + v[1][q];
                        hi = hi * kOzBaseI + v[2][q];
#pragma unroll
                        for (int d = 4; d < S; ++d) lo = lo * kOzBaseI + v[d][q];
                        val8[q] = (double)hi + (double)lo * lo_w;
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty + buf);
                if (CM == 0 && pairs) {
                    // element pair row m of tile pair (pI, pJ): t = 128 (mt % 8) + lrow -> (i, j) = (t % 32, t / 32)
                    const int m = mt * kOzBM + lrow;
                    const int t = m & 1023, pi = t & 31, pj = t >> 5;
                    const int ri = pI * 32 + pi, cj = pJ * 32 + pj, nn = out.pair_n;
                    const bool ok = ri < nn && cj < nn, diag = pI == pJ;
                    const double ra = pow2(ea_nx) * kOzScale;
                    {
                        const int un = next_u(u);
                        ea_nx = un < ue ? ea[unit_mt(un) * kOzBM + lrow] : 0;
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (q >= live) break;  // warp-uniform
                        const int col = nt * BN + c0 + q, x = col >> 1;
                        double w = val8[q] * ra * xchg[col];
                        if (diag && pi == pj) w += xchg[kOzBN + x];
                        double* o = out.c + (int64_t)x * out.ldc;
                        if (!(col & 1)) {  // W_x[32I + i, 32J + j]: lanes along rows 32I + i
                            if (ok) {
                                __stcs(o + (int64_t)cj * nn + ri, w);
                                if (out.rmax) atomicMax(psm + x * 32 + pi, (unsigned long long)__double_as_longlong(fabs(w)));
                            }
                        } else if (!diag) {  // the mirror W_x[32J + j, 32I + i]; row 32J + j is warp-uniform
                            if (ok) __stcs(o + (int64_t)ri * nn + cj, w);
                            if (out.rmax) {
                                const unsigned hw =
                                    (unsigned)((unsigned long long)__double_as_longlong(ok ? fabs(w) : 0.0) >> 32);
                                const unsigned mx = __reduce_max_sync(0xffffffffu, hw);
                                if (lane == 0 && mx) atomicMax(psm + 1024 + x * 32 + pj, (unsigned long long)mx << 32);
                            }
                        }
                    }
                    continue;
                }
                double ra = 0.0;
                if (CM == 0 && BN != kOzBN) {  // this unit's row exponent (prefetched), the next unit's load
                    ra = pow2(ea_nx) * kOzScale;
                    const int un = next_u(u);
                    ea_nx = un < ue ? ea[unit_mt(un) * kOzBM + lrow] : 0;
                }
                if (live <= 0) continue;
                const int m = mt * kOzBM + lrow;
                const int bm = m / out.mp, i = m - bm * out.mp;
                if (i >= out.mv) continue;
                if (!(CM == 0 && BN != kOzBN)) ra = pow2(ea[m]) * kOzScale;
                double* cb = out.c + (int64_t)bm * out.sc + i;
                const int* ebt = eb + nt * BN + c0;
                const double* sct = xchg + nt * BN + c0;  // 2^e_n of these columns (narrow forms)
                if (chunk) {
                    const int ibs = out.rn / kOzBM, rj = mt / ibs, ib = mt - rj * ibs, ri = ib * kOzBM + lrow;
                    if (ib != rib) {
                        flush_rmax(live);
                        rib = ib;
#pragma unroll
                        for (int q = 0; q < 8; ++q) rmx[q] = 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (q >= live) break;
                        double y = val8[q] * ra * (BN != kOzBN ? sct[q] : pow2(ebt[q]));
                        if (ri == rj) y += BN != kOzBN ? xchg[kOzBN + c0 + q] : out.dg[c0 + q];  // the c_0 I term
                        rmx[q] = fmax(rmx[q], fabs(y));
                        __stcs(cb + (int64_t)(c0 + q) * out.ldc, y);
                    }
                    continue;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (q >= live) break;
                    __stcs(cb + (int64_t)(nt * BN + c0 + q) * out.ldc,
                           val8[q] * ra * (BN != kOzBN ? sct[q] : pow2(ebt[q])));
                }
                continue;
            }
            if constexpr (BN == kOzBN) {
            // exact integer fold per column: hi = sum_{d<=4} acc_d 254^(4-d), lo = sum_{d>=5}
            // acc_d 254^(S+1-d); val = hi + lo 254^-(S-3). TMEM is drained 8 columns at a time, all S
            // accumulators in flight per wait.
            double val[kOzEC];
#pragma unroll
            for (int g8 = 0; g8 < kOzEC / 8; ++g8) {
                // all S accumulators of 8 columns in flight, one wait
                int32_t v[S][8];
#pragma unroll
                for (int d = 0; d < S; ++d) tmem_ld8(lane_addr + (uint32_t)(d * kOzBN + g8 * 8), v[d]);
                tmem_wait_ld();
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    long long hi = v[0][q], lo = v[3][q];
                    hi = hi * kOzBaseI + v[1][q];
                    hi = hi * kOzBaseI + v[2][q];
#pragma unroll
                    for (int d = 4; d < S; ++d) lo = lo * kOzBaseI + v[d][q];
                    val[g8 * 8 + q] = (double)hi + (double)lo * lo_w;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty + buf);
            // value = (hi + lo 254^-(S-3)) * 4 * 254^-4 * 2^e_r * 2^e_n
            const int m = mt * kOzBM + lrow;
            if (CM == 2) {
                // Z_kk[i, col] for this thread's 32 columns: Gram partials + base-254 digits. The row
                // kk = 2L-1 (Z_-L) of each signal row i in the tile is published through shared
                // memory for the <Z_-L, Z_k> partials (one named barrier of the 8 epilogue warps).
                const int i = m / out.tp2, kk = m - i * out.tp2, il = lrow / out.tp2;
                const bool row_ok = i < out.n;
                const double ra = pow2(ea[m]) * kOzScale;
                const int* ebt = eb + nt * kOzBN + h * kOzEC;
                double* xs = xchg + (tcount & 1) * 128 + il * 64 + h * kOzEC;
#pragma unroll
                for (int c = 0; c < kOzEC; ++c) {
                    const int col = nt * kOzBN + h * kOzEC + c;
                    val[c] = (row_ok && col < out.nv) ? val[c] * ra * pow2(ebt[c]) : 0.0;
                    if (kk == 2 * out.l - 1) xs[c] = val[c];
                }
                asm volatile("bar.sync 1, %0;" ::"n"(32 * kOzEpiWarps) : "memory");
                if (row_ok) {
                    // n % 64 == 0: position p = 2i + comp + 2n j has the same (p & 127) for every j,
                    // so the digit address of column pair j is base(comp) + j * jstride.
                    using YC = OzCfg<kOzZDigits>;
                    constexpr int kDig = kOzBM * YC::bk;  // bytes between the digit planes of a block
                    const int rr0 = (2 * i) & 127, pt0 = (2 * i) >> 7;
                    const int64_t jstride = (int64_t)(2 * out.n / 128) * out.kbz * kOzZDigits * kDig;
                    const int64_t kofs = (int64_t)(kk / YC::bk) * kOzZDigits * kDig + ((kk % YC::bk) >> 4) * 128 + (kk & 15);
                    int8_t* base0 = out.zd + (int64_t)pt0 * out.kbz * kOzZDigits * kDig + kofs +
                                    (rr0 >> 3) * YC::sbo + (rr0 & 7) * 16;
                    int8_t* base1 = out.zd + (int64_t)pt0 * out.kbz * kOzZDigits * kDig + kofs +
                                    ((rr0 + 1) >> 3) * YC::sbo + ((rr0 + 1) & 7) * 16;
                    const int j0 = (nt * kOzBN + h * kOzEC) >> 1;
#pragma unroll
                    for (int c2 = 0; c2 < kOzEC / 2; ++c2) {
                        const int j = j0 + c2;
                        if (2 * j >= out.nv) continue;
                        const int64_t p = ((int64_t)i + (int64_t)j * out.n) * 2;
                        const double2 xv = *reinterpret_cast<const double2*>(out.x + p);
                        const double2 cv = *reinterpret_cast<const double2*>(out.xc + p);
                        const double v0 = val[2 * c2], v1 = val[2 * c2 + 1];
                        gacc[0] = fma(xv.x, v0, fma(xv.y, v1, gacc[0]));
                        gacc[1] = fma(cv.x, v0, fma(cv.y, v1, gacc[1]));
                        gacc[2] = fma(xs[2 * c2], v0, fma(xs[2 * c2 + 1], v1, gacc[2]));
                        const double sc = pow2(-out.epos[j] - 1);
                        double r0 = v0 * sc, r1 = v1 * sc;  // |r| < 1/2
                        int8_t* d0 = base0 + j * jstride;
                        int8_t* d1 = base1 + j * jstride;
#pragma unroll
                        for (int t = 0; t < kOzZDigits; ++t) {
                            const double y0 = r0 * kOzBase, y1 = r1 * kOzBase;
                            const double t0 = y0 + kOzMagic, t1 = y1 + kOzMagic;  // rint in the low word
                            r0 = y0 - (t0 - kOzMagic);
                            r1 = y1 - (t1 - kOzMagic);
                            d0[t * kDig] = (int8_t)__double2loint(t0);
                            d1[t * kDig] = (int8_t)__double2loint(t1);
                        }
                    }
                }
                continue;
            }
            if (CM == 3) {
                // Y_a[p] = (C Z)[p, a] + c_0(a) X[p]; loss partial per order
                const int64_t p = m;
                if (p < out.count) {
                    const double ra = pow2(out.epos[m / (2 * out.n)]) * kOzScale;
                    const int* ebt = eb + nt * kOzBN + h * kOzEC;
                    const double xp = out.x[p], xcp = out.xc[p];
#pragma unroll
                    for (int c = 0; c < kOzEC; ++c) {
                        const int a = nt * kOzBN + h * kOzEC + c;
                        if (a < out.nv) {
                            const double yv = fma(out.c0[(int64_t)a * out.c0s], xp, val[c] * ra * pow2(ebt[c]));
                            if (out.c) __stcs(out.c + (int64_t)a * out.count + p, yv);
                            const double r = yv - xcp;
                            lacc[c] = fma(r, r, lacc[c]);
                        }
                    }
                }
                continue;
            }
            const int bm = m / out.mp, i = m - bm * out.mp;
            if (i < out.mv) {
                const double ra = pow2(ea[m]) * kOzScale;
                double* cb = out.c + (int64_t)bm * out.sc;
                const int* ebt = eb + nt * kOzBN + h * kOzEC;
#pragma unroll
                for (int c = 0; c < kOzEC; c += 2) {
                    const int n = nt * kOzBN + h * kOzEC + c;
                    if (n >= out.nv) break;
                    double v0 = val[c] * ra * pow2(ebt[c]);
                    double v1 = val[c + 1] * ra * pow2(ebt[c + 1]);
                    if (CM == 1 && out.dx) {  // the c_0 I term the synthesis left out: + c_0 X[i, j]
                        const double d = out.dgc[(int64_t)bm * out.dgs];
                        const double2 xv = *reinterpret_cast<const double2*>(out.dx + (i + (int64_t)(n >> 1) * out.ldc) * 2);
                        v0 = fma(d, xv.x, v0);
                        v1 = fma(d, xv.y, v1);
                    }
                    if (CM == 1 && fmse) {  // fused MSE: Y tile (even unit) / its dY tile (odd unit)
                        const int64_t o = (i + (int64_t)(n >> 1) * out.ldc) * 2;
                        const double2 xc = *reinterpret_cast<const double2*>(out.lxc + o);
                        if (!(u & 1)) {
                            *reinterpret_cast<double2*>(cb + o) = make_double2(v0, v1);  // re-read by this thread
                            const double rx = v0 - xc.x, ry = v1 - xc.y;
                            ls1 = fma(rx, rx, fma(ry, ry, ls1));
                        } else {
                            const double2 yv = *reinterpret_cast<const double2*>(
                                out.c + (int64_t)(bm - (mhalf * kOzBM) / out.mp) * out.sc + o);
                            ls2 = fma(yv.x - xc.x, v0, fma(yv.y - xc.y, v1, ls2));
                        }
                        continue;
                    }
                    if (CM == 0) {
                        const int64_t o0 = (int64_t)bm * out.sc + i + (int64_t)n * out.ldc;
                        __stcs(cb + i + (int64_t)n * out.ldc, v0);
                        if (n + 1 < out.nv) __stcs(cb + i + (int64_t)(n + 1) * out.ldc, v1);
                        for (int q = 0; q < out.npeers; ++q) {  // fused all-gather: peer copies
                            out.peers[q][o0] = v0;
                            if (n + 1 < out.nv) out.peers[q][o0 + out.ldc] = v1;
                        }
                    } else if (out.scw > 0) {  // fused reduce-scatter: the owner's receive slot
                        const int j = n >> 1, ho = j / out.scw;
                        double* d = out.dest[ho] + (int64_t)bm * out.ssc + (i + (int64_t)(j - ho * out.scw) * out.sld) * 2;
                        *reinterpret_cast<double2*>(d) = make_double2(v0, v1);
                    } else {
                        const int64_t o = (int64_t)bm * out.sc + (i + (int64_t)(n >> 1) * out.ldc) * 2;
                        __stcs(reinterpret_cast<double2*>(cb + (i + (int64_t)(n >> 1) * out.ldc) * 2), make_double2(v0, v1));
                        for (int q = 0; q < out.npeers; ++q)
                            *reinterpret_cast<double2*>(out.peers[q] + o) = make_double2(v0, v1);
                    }
                }
            }
            if (CM == 1 && fmse && (u & 1)) {  // pair unit done: warp sums in fixed order
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    ls1 += __shfl_xor_sync(0xffffffffu, ls1, o);
                    ls2 += __shfl_xor_sync(0xffffffffu, ls2, o);
                }
                if (lane == 0)
                    *reinterpret_cast<double2*>(out.lpart + ((int64_t)((mt - mhalf) * ntiles + nt) * kOzEpiWarps + ew) * 2) =
                        make_double2(ls1, ls2);
                ls1 = ls2 = 0.0;
            }
            }  // BN == kOzBN
        }
        if (chunk) flush_rmax(min((out.nv + 3) >> 2, out.nv - h * ((out.nv + 3) >> 2)));
        if (CM == 0 && pairs && BN != kOzBN && tcount > 0 && out.rmax) pair_flush(pI, pJ);
        if (CM == 1 && out.scw > 0) __threadfence_system();  // peer stores visible before the barrier
        if (CM == 2) {
            double* gp = out.part + (((int64_t)blockIdx.x * kOzEpiQ + h) * kOzBM + lrow) * 3;
            gp[0] = gacc[0];
            gp[1] = gacc[1];
            gp[2] = gacc[2];
        }
        if (CM == 3) {
#pragma unroll
            for (int c = 0; c < kOzEC; ++c) {
                double v = lacc[c];
#pragma unroll
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                lacc[c] = v;
            }
            if (lane == 0) {
                double* lp = out.part + (((int64_t)blockIdx.x * kOzEpiQ + h) * 4 + lg) * kOzEC;
#pragma unroll
                for (int c = 0; c < kOzEC; ++c) lp[c] = lacc[c];
            }
        }
    }
    tc_fence_before();
    if (CL > 1) cluster_sync_all(); else __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------- INT8 tensor-core synthesis
//
// Q(a) = c_0 I + sum_k c_k P_k + c_-k P_k^T (and dQ/da with c'_k) for one tile pair {(I,J),(J,I)}
// as a GEMM whose rows are ELEMENT PAIRS and whose K is the power index: row t of a pair holds the
// powers of element e = (32I+i, 32J+j) in K [0, kh) and of its mirror e' = (32J+j, 32I+i) in
// K [kh, 2 kh) (OzView mode 7: 5 base-254 digits, one exponent per row over all 2L values -- the
// same ~2^-40 quantisation as the packed cache). B = per operator row two coefficient rows
// [c_k | c_-k] and [c_-k | c_k] (6 digits, one 16-row tile loaded once per CTA), so accumulator
// column 2x is Q_x[e] and column 2x + 1 is Q_x[e'] -- every thread owns both outputs of its row,
// with no exchange between threads. The multiply-adds run on the tensor cores; the SMs stream
// digits (TMA ring) and run a short fold per element, so the synthesis of one row shell can share
// the GPU with the product GEMM of the previous one (capi.cu packed_products). One CTA per SM
// walks whole pairs (8 M tiles of 128 rows): warp 0 = TMA producer, warps 1-2 = MMA issuers, then G
// epilogue groups of 4 warps taking tiles round robin (TMEM: 4 accumulator buffers, 128 columns
// apart, each 6 digit sums x 16 columns).
constexpr int kDsBN = 16;
constexpr int kDsSA = 5, kDsSB = 6;
constexpr int kDsNB = 4;
constexpr int kDsIssuers = 2;                  // MMA-issuing warps (kDsNB % kDsIssuers == 0); dbg & 2: 1
constexpr int kDsAStage = kDsSA * kOzBM * 64;  // one M tile x one 64-byte K block (40 KB)
constexpr int kDsTiles = 8;                    // M tiles per pair (1024 element pairs / 128)

__host__ __device__ constexpr int ds_b_bytes(int kp) { return kDsSB * kDsBN * kp; }
__host__ __device__ constexpr int ds_fixed_bytes(int kp) { return ds_b_bytes(kp) + 256; }  // B + barriers
static int ds_stages(int kp) {
    static const int forced = [] {
        const char* e = std::getenv("FGFRFT_DS_STAGES");
        return e ? std::atoi(e) : 0;
    }();
    int st = (227 * 1024 - ds_fixed_bytes(kp)) / kDsAStage;
    if (forced > 0 && forced < st) st = forced;
    return st > 5 ? 5 : st;
}
static int ds_smem(int kp) { return ds_stages(kp) * kDsAStage + ds_fixed_bytes(kp); }

template <int W>
__device__ __forceinline__ void tmem_ldw(uint32_t taddr, int32_t (&v)[W]) {
    if constexpr (W == 2) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(taddr));
    } else if constexpr (W == 4) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(taddr));
    } else {
        static_assert(W == 8, "2, 4 or 8 columns");
        tmem_ld8(taddr, v);
    }
}

// c_x(s k) of table row x (c_k at l_used + k), 0 beyond the truncation
__device__ __forceinline__ double ds_coef(const double* coef, int coef_ld, int l_used, int x, int k) {
    return (k <= l_used && k >= -l_used) ? coef[(size_t)x * coef_ld + l_used + k] : 0.0;
}

// B operand: row 2x = [c_x(k) | c_x(-k)], row 2x + 1 = [c_x(-k) | c_x(k)] (K halves of kh = kp / 2,
// k = kk + 1), the canonical K-major layout of a 16-row tile with 64-byte K blocks.
__global__ void __launch_bounds__(512) dsynth_coef_kernel(const double* __restrict__ coef, int coef_ld, int l_used,
                                                          int ac, int kp, int8_t* __restrict__ bd, int* __restrict__ eb) {
    __shared__ unsigned long long mx[kDsBN];
    const int kh = kp / 2, runs = kp / 16;  // one thread per (row, 16-byte K run)
    const int r = threadIdx.x / runs, q = threadIdx.x - r * runs;
    if (threadIdx.x < kDsBN) mx[threadIdx.x] = 0ull;
    double x[16];
    double m = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int kk = q * 16 + i;
        const bool hi = kk >= kh;
        const int k = (hi ? kk - kh : kk) + 1;
        const bool neg = hi != (bool)(r & 1);
        x[i] = r < 2 * ac ? ds_coef(coef, coef_ld, l_used, r >> 1, neg ? -k : k) : 0.0;
        m = fmax(m, fabs(x[i]));
    }
    __syncthreads();
    if (m > 0.0) atomicMax(mx + r, (unsigned long long)__double_as_longlong(m));
    __syncthreads();
    const double rm = __longlong_as_double((long long)mx[r]);
    int e = 0;
    if (rm > 0.0) frexp(rm, &e);
    if (q == 0) eb[r] = e;
    const double sc = rm > 0.0 ? pow2(-e - 1) : 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] *= sc;
    const int k0 = q * 16, kb = k0 / 64, cl = (k0 >> 4) & 3;
    int8_t* base = bd + (int64_t)kb * kDsSB * kDsBN * 64 + (r >> 3) * 512 + cl * 128 + (r & 7) * 16;
#pragma unroll
    for (int s2 = 0; s2 < kDsSB; ++s2) {
        uint32_t w[4];
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
            uint32_t packed = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const double y = x[qq * 4 + i] * kOzBase;
                const double tt = y + kOzMagic;
                x[qq * 4 + i] = y - (tt - kOzMagic);
                packed |= ((uint32_t)__double2loint(tt) & 0xFFu) << (8 * i);
            }
            w[qq] = packed;
        }
        *reinterpret_cast<uint4*>(base + s2 * kDsBN * 64) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// max of non-negative doubles over the warp by their high words (sign, exponent, 20 mantissa
// bits): the slicer only takes the exponent of a row max, which the high word fixes exactly
__device__ __forceinline__ unsigned long long ds_warp_max_hi(double v) {
    const unsigned h = (unsigned)((unsigned long long)__double_as_longlong(v) >> 32);
    return (unsigned long long)__reduce_max_sync(0xffffffffu, h) << 32;
}

template <int AC, int G>
__global__ void __launch_bounds__(32 * (1 + kDsIssuers + 4 * G), 1)
dsynth_kernel(const int8_t* __restrict__ a, const int* __restrict__ ea, const int8_t* __restrict__ b,
              const int* __restrict__ eb, int kblocks, int stages, int n, int nt, int p0, int p1,
              const double* __restrict__ coef, int coef_ld, int l_used, double* __restrict__ out, int64_t ostride,
              unsigned long long* __restrict__ rowmax, int64_t mp, int dbg, int nodiag) {
    constexpr int W = 2 * AC;        // live B rows / accumulator columns
    constexpr int TPG = kDsTiles / G;  // tiles of a pair per epilogue group
    static_assert(kDsTiles % G == 0, "groups divide the tiles of a pair");
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* sa = smem;
    unsigned char* sb = smem + (size_t)stages * kDsAStage;
    uint64_t* full = reinterpret_cast<uint64_t*>(sb + ds_b_bytes(kblocks * 64));
    uint64_t* empty = full + 5;
    uint64_t* tfull = empty + 5;  // [NB]
    uint64_t* tempty = tfull + kDsNB;
    uint64_t* bfull = tempty + kDsNB;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t pstart = p0 + blockIdx.x;
    const int tile_kb = kblocks;  // K blocks per M tile
    const int nis = (dbg & 2) ? 1 : kDsIssuers;  // MMA issuers
    const int sr = stages / nis;                 // stages per issuer ring
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int u = 0; u < kDsNB; ++u) {
            mbar_init(tfull + u, 1);
            mbar_init(tempty + u, 4);
        }
        mbar_init(bfull, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();  // the digits are read once per step (dsynth)
            mbar_arrive_expect_tx(bfull, (uint32_t)ds_b_bytes(kblocks * 64));
            bulk_g2s(sb, b, (uint32_t)ds_b_bytes(kblocks * 64), bfull);
            // one stage ring per MMA issuer (issuer w consumes tiles w, w + nis, ...): a ring whose
            // stages alternated between issuers would let one wait on a phase two ahead (parity alias)
            int itr[kDsIssuers] = {};
            int tcount = 0;
            for (int64_t p = pstart; p < p1; p += gridDim.x) {
                const unsigned char* ga = reinterpret_cast<const unsigned char*>(a) + p * kDsTiles * (int64_t)tile_kb * kDsAStage;
                for (int sub = 0; sub < kDsTiles; ++sub, ++tcount) {  // a pair's tiles are contiguous
                    const int r = tcount % nis;
                    for (int kb = 0; kb < tile_kb; ++kb) {
                        const int it = itr[r]++;
                        const int s = r * sr + it % sr;
                        if (it >= sr) mbar_wait(empty + s, ((it / sr) - 1) & 1);
                        mbar_arrive_expect_tx(full + s, kDsAStage);
                        bulk_g2s_hint(sa + (size_t)s * kDsAStage, ga + ((int64_t)sub * tile_kb + kb) * kDsAStage, kDsAStage,
                                      full + s, pol);
                    }
                }
            }
        }
    } else if (warp <= kDsIssuers) {
        // MMA issuers: one tcgen05.mma costs its issuing thread ~75 cycles whatever N (measured,
        // tools/probes/mma_probe.cu), more than the tensor pipe needs for these N <= 96 tiles, so
        // kDsIssuers warps issue alternate tiles (issuer w: tiles w, w + kDsIssuers, ...)
        const int me = warp - 1;
        if (lane == 0 && me < nis) {
            mbar_wait(bfull, 0);
            tc_fence_after();
            const uint32_t b0 = smem_u32(sb);
            int it = 0, tcount = 0;
            for (int64_t p = pstart; p < p1; p += gridDim.x)
                for (int sub = 0; sub < kDsTiles; ++sub, ++tcount) {
                    if (tcount % nis != me) continue;
                    const int buf = tcount % kDsNB;
                    if (tcount >= kDsNB) mbar_wait(tempty + buf, ((tcount / kDsNB) - 1) & 1);
                    tc_fence_after();
                    const uint32_t acc = tmem + (uint32_t)buf * 128;
                    for (int kb = 0; kb < tile_kb; ++kb, ++it) {
                        const int s = me * sr + it % sr;
                        mbar_wait(full + s, (it / sr) & 1);
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(sa + (size_t)s * kDsAStage);
                        if (!(dbg & 1))
#pragma unroll
                            for (int j = 0; j < 2; ++j)
#pragma unroll
                                for (int t = 1; t <= kDsSA; ++t) {
                                    // A digit t x B digits 1 .. 7 - t -> digit sums t - 1 .. 5 (columns 16 (t-1) ..)
                                    const uint64_t ad = umma_desc(a0 + (t - 1) * kOzBM * 64 + j * 256, 128, 512);
                                    const uint64_t bd = umma_desc(b0 + kb * kDsSB * kDsBN * 64 + j * 256, 128, 512);
                                    mma_i8(acc + (uint32_t)((t - 1) * kDsBN), ad, bd,
                                           idesc_i8(kOzBM, (kDsSB + 1 - t) * kDsBN), (kb > 0 || j > 0 || t > 1) ? 1u : 0u);
                                }
                        mma_commit(empty + s);
                    }
                    mma_commit(tfull + buf);
                }
        }
    } else {
        const int grp = (warp - 1 - kDsIssuers) >> 2, lg = warp & 3;
        const int lrow = lg * 32 + lane;
        int ebv[W];
        double c0v[AC];
#pragma unroll
        for (int c = 0; c < W; ++c) ebv[c] = eb[c];
#pragma unroll
        for (int x = 0; x < AC; ++x) c0v[x] = nodiag ? 0.0 : coef[(size_t)x * coef_ld + l_used];  // nodiag: Q - c_0 I
        constexpr double w1 = 1.0 / 254.0, w2 = w1 * w1, w3 = w2 * w1, w4 = w3 * w1, w5 = w4 * w1;
        // this group's tiles of a pair are sub = G q + grp; their row exponents are loaded one pair
        // ahead (a DRAM round trip under load is ~1-2 us)
        int eaq[TPG], ean[TPG];
        auto load_ea = [&](int64_t pp, int (&dst)[TPG]) {
#pragma unroll
            for (int q2 = 0; q2 < TPG; ++q2)
                dst[q2] = pp < p1 ? __ldcs(ea + (pp * kDsTiles + G * q2 + grp) * kOzBM + lrow) : 0;
        };
        load_ea(pstart, eaq);
        int jp = 0;
        for (int64_t p = pstart; p < p1; p += gridDim.x, ++jp) {
            load_ea(p + gridDim.x, ean);
            int I, J;
            pair_of_imajor((int)p, nt, I, J);
            const bool diag = I == J;
            const int i = lane, ri = I * kTile + i;  // this thread's row of Q_IJ (fixed over the pair)
            double rij[AC];
#pragma unroll
            for (int x = 0; x < AC; ++x) rij[x] = 0.0;
#pragma unroll
            for (int q2 = 0; q2 < TPG; ++q2) {
                const int sub = G * q2 + grp, tcount = jp * kDsTiles + sub;
                const int buf = tcount % kDsNB;
                const int j = 4 * sub + lg;  // t = 128 sub + 32 lg + lane = i + 32 j
                const double ra = pow2(eaq[q2]) * (4.0 / (254.0 * 254.0));  // 2^2 x 254^-2: f = sum v_d 254^-d
                mbar_wait(tfull + buf, (tcount / kDsNB) & 1);
                tc_fence_after();
                int32_t v[6][W];
#pragma unroll
                for (int d = 0; d < 6; ++d)
                    tmem_ldw<W>(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(buf * 128 + d * kDsBN), v[d]);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty + buf);
                const int cj = J * kTile + j;
                const bool ok = ri < n && cj < n;
#pragma unroll
                for (int x = 0; x < AC; ++x) {
                    double val[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int c = 2 * x + h;  // |v| < 2^31: exact in double; 6 roundings ~ 2^-51 relative
                        double f = fma((double)v[5][c], w5, (double)v[4][c] * w4);
                        f = fma((double)v[3][c], w3, f);
                        f = fma((double)v[2][c], w2, f);
                        f = fma((double)v[1][c], w1, f);
                        f += (double)v[0][c];
                        val[h] = f * ra * pow2(ebv[c]);
                        if (diag && i == j) val[h] += c0v[x];
                    }
                    double* o = out + x * ostride;
                    if (ok) {
                        __stcs(o + (int64_t)cj * n + ri, val[0]);  // Q[32I+i, 32J+j]: lanes along rows
                        rij[x] = fmax(rij[x], fabs(val[0]));
                    }
                    if (!diag) {  // Q[32J+j, 32I+i]; row 32J+j's max over this warp's 32 columns
                        if (ok) __stcs(o + (int64_t)ri * n + cj, val[1]);
                        const unsigned long long m = ds_warp_max_hi(ok ? fabs(val[1]) : 0.0);
                        if (lane == 0 && m && cj < n) atomicMax(rowmax + (int64_t)x * mp + cj, m);
                    }
                }
            }
#pragma unroll
            for (int x = 0; x < AC; ++x)
                if (ri < n && rij[x] > 0.0)
                    atomicMax(rowmax + (int64_t)x * mp + ri, (unsigned long long)__double_as_longlong(rij[x]));
#pragma unroll
            for (int q2 = 0; q2 < TPG; ++q2) eaq[q2] = ean[q2];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------- host launchers

int oz_slices_default() { return 6; }

int oz_zdigits() { return kOzZDigits; }

int oz_bk(int slices) { return slices <= 6 ? OzCfg<6>::bk : OzCfg<7>::bk; }

size_t oz_operand_bytes(int slices, int64_t rows_padded, int64_t kp) { return (size_t)slices * rows_padded * kp; }

cudaError_t launch_oz_slice(const OzView& v, int slices, int tr, int8_t* dst, int* exps, unsigned long long* rowmax,
                            cudaStream_t stream) {
    const int rows = v.nb * v.rp;
    if (rows % 64 || v.kp % 64 || v.rp % tr) return cudaErrorInvalidValue;
    if (!v.tiled && !v.rfast && v.ra == 1 && v.ka == 0 && v.ks == 2 && v.rv % 2 == 0 && v.nb == 1) {
        // complex signal columns (re / im row pairs): one fused pass
        const unsigned blocks = (unsigned)(rows / 2);
        if (slices == 7)
            oz_rowslice_pairs_kernel<7><<<blocks, 64, 0, stream>>>(v, tr, dst, exps);
        else if (slices == 8)
            oz_rowslice_pairs_kernel<8><<<blocks, 64, 0, stream>>>(v, tr, dst, exps);
        else if (slices == 6)
            oz_rowslice_pairs_kernel<6><<<blocks, 64, 0, stream>>>(v, tr, dst, exps);
        else if (slices == 5)
            oz_rowslice_pairs_kernel<5><<<blocks, 64, 0, stream>>>(v, tr, dst, exps);
        else
            return cudaErrorInvalidValue;
        return cudaGetLastError();
    }
    if (!v.tiled && v.rfast && rows / 32 >= 2 * FGFRFT_SMS) {  // tall: one fused pass
        if (slices == 7)
            oz_rowslice_direct_kernel<7><<<rows / 32, 256, 0, stream>>>(v, tr, dst, exps);
        else if (slices == 8)
            oz_rowslice_direct_kernel<8><<<rows / 32, 256, 0, stream>>>(v, tr, dst, exps);
        else if (slices == 6)
            oz_rowslice_direct_kernel<6><<<rows / 32, 256, 0, stream>>>(v, tr, dst, exps);
        else if (slices == 5)
            oz_rowslice_direct_kernel<5><<<rows / 32, 256, 0, stream>>>(v, tr, dst, exps);
        else
            return cudaErrorInvalidValue;
        return cudaGetLastError();
    }
    cudaError_t e = cudaMemsetAsync(rowmax, 0, (size_t)rows * sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return e;
    dim3 grid(rows / 64, v.kp / 64);
    if (!v.tiled && v.rfast) {
        oz_rowmax_direct_kernel<<<grid, 64, 0, stream>>>(v, rowmax);
        if (slices == 7)
            oz_slice_direct_kernel<7><<<grid, 64, 0, stream>>>(v, rowmax, tr, dst, exps);
        else if (slices == 8)
            oz_slice_direct_kernel<8><<<grid, 64, 0, stream>>>(v, rowmax, tr, dst, exps);
        else if (slices == 6)
            oz_slice_direct_kernel<6><<<grid, 64, 0, stream>>>(v, rowmax, tr, dst, exps);
        else if (slices == 5)
            oz_slice_direct_kernel<5><<<grid, 64, 0, stream>>>(v, rowmax, tr, dst, exps);
        else
            return cudaErrorInvalidValue;
        return cudaGetLastError();
    }
    oz_rowmax_kernel<<<grid, 256, 0, stream>>>(v, rowmax);
    if (slices == 5)  // the synthesis digit cache (dsynth_kernel)
        oz_slice_kernel<5><<<grid, 256, 0, stream>>>(v, rowmax, tr, dst, exps);
    else if (slices == 7)
        oz_slice_kernel<7><<<grid, 256, 0, stream>>>(v, rowmax, tr, dst, exps);
    else if (slices == 8)
        oz_slice_kernel<8><<<grid, 256, 0, stream>>>(v, rowmax, tr, dst, exps);
    else if (slices == 6)
        oz_slice_kernel<6><<<grid, 256, 0, stream>>>(v, rowmax, tr, dst, exps);
    else
        return cudaErrorInvalidValue;
    return cudaGetLastError();
}

// Digits only, from row maxima already in `rowmax` (e.g. left by the node-operator GEMM).
cudaError_t launch_oz_slice_ready(const OzView& v, int slices, int tr, int8_t* dst, int* exps,
                                  const unsigned long long* rowmax, cudaStream_t stream) {
    const int rows = v.nb * v.rp;
    if (rows % 64 || v.kp % 64 || v.rp % tr) return cudaErrorInvalidValue;
    dim3 grid(rows / 64, v.kp / 64);
    const bool direct = !v.tiled && v.rfast;
#define FGB_SL(S_)                                                                                  \
    if (slices == S_) {                                                                             \
        if (direct)                                                                                 \
            oz_slice_direct_kernel<S_><<<grid, 64, 0, stream>>>(v, rowmax, tr, dst, exps);          \
        else                                                                                        \
            oz_slice_kernel<S_><<<grid, 256, 0, stream>>>(v, rowmax, tr, dst, exps);                \
        return cudaGetLastError();                                                                  \
    }
    FGB_SL(5)
    FGB_SL(6)
    FGB_SL(7)
    FGB_SL(8)
#undef FGB_SL
    return cudaErrorInvalidValue;
}

template <int S, int CM, int CL, int BN = kOzBN, bool P = false>
static cudaError_t oz_launch_cl(const int8_t* a, const int* ea, int mtiles, const int8_t* b, const int* eb, int ntiles,
                                int kp, const OzOut& out, cudaStream_t stream) {
    static PerDeviceOnce attr;
    if (cudaError_t e = attr.run([] {
            return cudaFuncSetAttribute(ozgemm_kernel<S, CM, CL, BN, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (OzCfg<S, BN, P>::smem));
        }))
        return e;
    const int units = mtiles * (ntiles / CL);
    OzOut o2 = out;
    if (CM == 1 && BN == kOzBN) {
        // B bands: keep the B operand's band (evict_last) L2-resident beside the streaming A tiles
        static const int forced_bands = [] {
            const char* e = std::getenv("FGFRFT_OZ_BANDS");
            return e ? std::atoi(e) : 0;
        }();
        const int ngroups = ntiles / CL;
        const double bbytes = (double)ntiles * BN * kp * S, cap = 56e6;
        int nb = forced_bands > 0 ? forced_bands : (bbytes > cap ? (int)((bbytes + cap - 1) / cap) : 1);
        while (nb < ngroups && ngroups % nb) ++nb;
        o2.nband = (nb >= 1 && nb <= ngroups && ngroups % nb == 0) ? nb : 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kOzThreads);
    cfg.dynamicSmemBytes = (OzCfg<S, BN, P>::smem);
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // persistent grid = the clusters that are co-resident (GPC sizes are not multiples of CL)
    static std::atomic<int> max_clusters_dev[64];
    int dev = 0;
    cudaGetDevice(&dev);
    int max_clusters = max_clusters_dev[dev & 63].load(std::memory_order_relaxed);
    if (max_clusters == 0) {
        cfg.gridDim = dim3(FGFRFT_SMS / CL * CL);
        int mc = 0;
        if (cudaOccupancyMaxActiveClusters(&mc, ozgemm_kernel<S, CM, CL, BN, P>, &cfg) != cudaSuccess || mc <= 0) {
            cudaGetLastError();
            mc = FGFRFT_SMS / CL;
        }
        max_clusters = mc;
        max_clusters_dev[dev & 63].store(mc, std::memory_order_relaxed);
    }
    if (out.max_ctas > 0 && out.max_ctas / CL < max_clusters) max_clusters = out.max_ctas / CL > 0 ? out.max_ctas / CL : 1;
    int clusters = units < max_clusters ? units : max_clusters;
    if (CM == 0 && CL == 1 && out.rmax && !out.pair_nt) {  // row-max mode: a multiple of the row blocks per column
        const int ibs = out.rn / kOzBM;
        if (clusters >= ibs) clusters = clusters / ibs * ibs;
    }
    cfg.gridDim = dim3(clusters * CL);
    return cudaLaunchKernelEx(&cfg, ozgemm_kernel<S, CM, CL, BN, P>, a, ea, b, eb, kp / OzCfg<S, BN, P>::bk, mtiles, ntiles, o2);
}

template <int S, int CM>
static cudaError_t oz_launch(const int8_t* a, const int* ea, int mrows, const int8_t* b, const int* eb, int nrows,
                             int kp, const OzOut& out, cudaStream_t stream) {
    const int mtiles = mrows / kOzBM, ntiles = nrows / kOzBN;
    static const int forced = [] {
        const char* e = std::getenv("FGFRFT_OZ_CLUSTER");
        return e ? std::atoi(e) : 0;
    }();
    // Measured on B200 (tools/bench_int8gemm.py): pairs win (3.13 vs 3.05 POPS unclustered);
    // clusters of 4 / 8 lose co-residency (GPC sizes) more than they save in L2 traffic.
    int cl = ntiles % 2 == 0 ? 2 : 1;
    if ((forced == 1 || forced == 2 || forced == 4 || forced == 8) && ntiles % forced == 0) cl = forced;
    switch (cl) {
        case 8: return oz_launch_cl<S, CM, 8>(a, ea, mtiles, b, eb, ntiles, kp, out, stream);
        case 4: return oz_launch_cl<S, CM, 4>(a, ea, mtiles, b, eb, ntiles, kp, out, stream);
        case 2: return oz_launch_cl<S, CM, 2>(a, ea, mtiles, b, eb, ntiles, kp, out, stream);
        default: return oz_launch_cl<S, CM, 1>(a, ea, mtiles, b, eb, ntiles, kp, out, stream);
    }
}

// Skinny CM 0 product (out.nv <= 32, no peers): B sliced with 32-row tiles (launch_oz_slice tr =
// kOzTileNarrow), nrows == 32; narrow TMEM accumulators, double-buffered.
cudaError_t launch_ozgemm_narrow(int slices, const int8_t* a, const int* ea, int mrows, const int8_t* b,
                                 const int* eb, int nrows, int kp, const OzOut& out, cudaStream_t stream) {
    // pair mode (out.pair_nt): up to 2 B tiles of 32 rows (2r <= 64 output columns)
    const int nt = nrows / kOzTileNarrow;
    if (mrows % kOzBM || nrows % kOzTileNarrow || kp % 64 || out.npeers ||
        (out.pair_nt ? (nt > 2 || out.nv > nrows || mrows % (8 * kOzBM)) : (nt != 1 || out.nv > kOzTileNarrow)))
        return cudaErrorInvalidValue;
    const int mtiles = mrows / kOzBM;
    if (out.pair_nt) {
        if (slices == 6) return oz_launch_cl<6, 0, 1, kOzTileNarrow, true>(a, ea, mtiles, b, eb, nt, kp, out, stream);
        return cudaErrorInvalidValue;
    }
    if (slices == 6) return oz_launch_cl<6, 0, 1, kOzTileNarrow>(a, ea, mtiles, b, eb, nt, kp, out, stream);
    if (slices == 7) return oz_launch_cl<7, 0, 1, kOzTileNarrow>(a, ea, mtiles, b, eb, nt, kp, out, stream);
    if (slices == 8) return oz_launch_cl<8, 0, 1, kOzTileNarrow>(a, ea, mtiles, b, eb, nt, kp, out, stream);
    return cudaErrorInvalidValue;
}

// C (from OzOut) = A_sliced (mrows x kp) * B_sliced (nrows x kp)^T; mrows % 128 == 0, nrows % 64 == 0.
cudaError_t launch_ozgemm_ex(int slices, int cm, const int8_t* a, const int* ea, int mrows, const int8_t* b,
                             const int* eb, int nrows, int kp, const OzOut& out, cudaStream_t stream) {
    if (mrows % kOzBM || nrows % kOzBN || kp % 64) return cudaErrorInvalidValue;
    if (cm <= 1 && out.mp <= 0) return cudaErrorInvalidValue;
#define FGB_OZ(S_)                                                                       \
    if (slices == S_) {                                                                  \
        switch (cm) {                                                                    \
            case 0: return oz_launch<S_, 0>(a, ea, mrows, b, eb, nrows, kp, out, stream); \
            case 1: return oz_launch<S_, 1>(a, ea, mrows, b, eb, nrows, kp, out, stream); \
            case 2: return oz_launch<S_, 2>(a, ea, mrows, b, eb, nrows, kp, out, stream); \
            case 3: return oz_launch<S_, 3>(a, ea, mrows, b, eb, nrows, kp, out, stream); \
            default: return cudaErrorInvalidValue;                                       \
        }                                                                                \
    }
    FGB_OZ(5)
    FGB_OZ(6)
    FGB_OZ(7)
    FGB_OZ(8)
#undef FGB_OZ
    return cudaErrorInvalidValue;
}

cudaError_t launch_ozgemm(int slices, int cm, const int8_t* a, const int* ea, int mrows, const int8_t* b,
                          const int* eb, int nrows, int kp, double* c, int64_t ldc, int64_t sc, int mv, int mp, int nv,
                          cudaStream_t stream, double* const* peers, int npeers, int max_ctas) {
    if (cm > 1 || npeers < 0 || npeers > 7) return cudaErrorInvalidValue;
    OzOut out;
    for (int q = 0; q < npeers; ++q) out.peers[q] = peers[q];
    out.npeers = npeers;
    out.c = c;
    out.ldc = ldc;
    out.sc = sc;
    out.mv = mv;
    out.mp = mp;
    out.nv = nv;
    out.max_ctas = max_ctas;
    return launch_ozgemm_ex(slices, cm, a, ea, mrows, b, eb, nrows, kp, out, stream);
}


size_t dsynth_cache_rows(int n) {
    const int64_t nt = ceil_div(n, kTile);
    return (size_t)(nt * (nt + 1) / 2) * kDsTiles * kOzBM;
}
int dsynth_slices() { return kDsSA; }
int dsynth_kp(int l) { return (int)(2 * ceil_div(l, 64) * 64); }
size_t dsynth_coef_bytes(int kp) { return (size_t)ds_b_bytes(kp) + kDsBN * sizeof(int); }

// The digit cache from the tiled FP64 slabs: OzView mode 7, 5 digits, 128-row tiles.
cudaError_t launch_dsynth_build(const double* slabs, int n, int l, int kp, int8_t* digits, int* exps,
                                unsigned long long* rowmax_tmp, cudaStream_t stream, int slices) {
    const int nt = (int)ceil_div(n, kTile);
    OzView v{slabs, 0, 0, (int64_t)nt * nt * kTileElems, 0, 0, (int)dsynth_cache_rows(n), (int)dsynth_cache_rows(n),
             1, kp, kp, true};
    v.tiled = 7;
    v.nt = nt;
    v.l = l;
    v.tp2 = n;
    return launch_oz_slice(v, slices > 0 ? slices : kDsSA, kOzBM, digits, exps, rowmax_tmp, stream);
}

// Coefficient digits for `ac` operator rows (table rows of width coef_ld, c_k at l_used + k) into
// bsl (dsynth_coef_bytes(kp): digits, then 16 exponents).
cudaError_t launch_dsynth_coefs(const double* coef, int coef_ld, int l_used, int ac, int kp, int8_t* bsl,
                                cudaStream_t stream) {
    if (ac != 1 && ac != 2 && ac != 4) return cudaErrorInvalidValue;
    dsynth_coef_kernel<<<1, kDsBN * (kp / 16), 0, stream>>>(coef, coef_ld, l_used, ac, kp, bsl,
                                             reinterpret_cast<int*>(bsl + ds_b_bytes(kp)));
    return cudaGetLastError();
}

template <int AC, int G>
static cudaError_t dsynth_launch(const int8_t* digits, const int* exps, const int8_t* bsl, int kp, int n, int p0,
                                 int p1, const double* coef, int coef_ld, int l_used, double* out, int64_t out_stride,
                                 unsigned long long* rowmax, int64_t mp, int max_ctas, cudaStream_t stream, int nodiag) {
    static PerDeviceOnce attr;
    const int smem = ds_smem(kp);
    if (cudaError_t e = attr.run([&] {
            return cudaFuncSetAttribute(dsynth_kernel<AC, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        }))
        return e;
    const int pairs = p1 - p0;
    int grid = FGFRFT_SMS;
    if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
    if (pairs < grid) grid = pairs;
    if (grid <= 0) return cudaSuccess;
    const int nt = (int)ceil_div(n, kTile);
    static const int dbg = [] {
        const char* e = std::getenv("FGFRFT_DS_DEBUG");  // timing experiments only: 1 = skip the MMAs
        return e ? std::atoi(e) : 0;
    }();
    dsynth_kernel<AC, G><<<grid, 32 * (1 + kDsIssuers + 4 * G), smem, stream>>>(
        digits, exps, bsl, reinterpret_cast<const int*>(bsl + ds_b_bytes(kp)), kp / 64, ds_stages(kp), n, nt, p0, p1,
        coef, coef_ld, l_used, out, out_stride, rowmax, mp, dbg, nodiag);
    return cudaGetLastError();
}

cudaError_t launch_dsynth(const int8_t* digits, const int* exps, const int8_t* bsl, int kp, int n, int p0, int p1,
                          const double* coef, int coef_ld, int l_used, int ac, double* out, int64_t out_stride,
                          unsigned long long* rowmax, int64_t mp, int max_ctas, cudaStream_t stream, int nodiag) {
    if (kp % 128 || kp > 512) return cudaErrorInvalidValue;
    if (p1 < 0) {
        const int64_t nt = ceil_div(n, kTile);
        p1 = (int)(nt * (nt + 1) / 2);
    }
    static const int groups = [] {
        const char* e = std::getenv("FGFRFT_DS_GROUPS");
        return e ? std::atoi(e) : 4;
    }();
    switch (ac * 10 + (groups == 2 ? 2 : 4)) {
        case 12: return dsynth_launch<1, 2>(digits, exps, bsl, kp, n, p0, p1, coef, coef_ld, l_used, out, out_stride, rowmax, mp, max_ctas, stream, nodiag);
        case 14: return dsynth_launch<1, 4>(digits, exps, bsl, kp, n, p0, p1, coef, coef_ld, l_used, out, out_stride, rowmax, mp, max_ctas, stream, nodiag);
        case 22: return dsynth_launch<2, 2>(digits, exps, bsl, kp, n, p0, p1, coef, coef_ld, l_used, out, out_stride, rowmax, mp, max_ctas, stream, nodiag);
        case 24: return dsynth_launch<2, 4>(digits, exps, bsl, kp, n, p0, p1, coef, coef_ld, l_used, out, out_stride, rowmax, mp, max_ctas, stream, nodiag);
        case 42:
        case 44: return dsynth_launch<4, 2>(digits, exps, bsl, kp, n, p0, p1, coef, coef_ld, l_used, out, out_stride, rowmax, mp, max_ctas, stream, nodiag);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fgb
