// oz.cuh -- host-visible interface of the Ozaki-scheme INT8 tensor-core GEMM (ozgemm.cu).
#pragma once
#include "common.cuh"

namespace fgb {

// Logical operand (R rows x K): element (r, k) of batch block bt sits at
//   src[bt * sbatch + (r >> ra) * rs + (r & ra) + (k >> ka) * ks + (k & ka)]
// or, for a tiled cache slab (tiled = 1 / 2), at the tiled position of P(r, k) / P(k, r).
// (ra / ka = 1 split a complex dimension into its (re, im) halves). Rows are grouped in batch
// blocks of rv valid rows padded to rp (a multiple of the tile rows); the sliced operand holds
// nb * rp rows. Padding rows / columns are zero.
struct OzView {
    const double* src;
    int64_t rs, ks, sbatch;
    int ra, ka;
    int rv, rp, nb;  // valid rows per block, padded rows per block, blocks
    int kv, kp;      // valid K, padded K (multiple of kOzBK)
    bool rfast;      // rows are the contiguous direction of the source
    int tiled = 0;   // 1: src is a tiled cache slab (common.cuh), element (r, k) = P(r, k);
                     // 2: the same slab read transposed, element (r, k) = P(k, r);
                     // 3: interleaved stacked cache, row r = i * tp2 + kk: term kk < L is
                     //    P_(kk+1)(i, k), L <= kk < 2L is P_(kk-L+1)(k, i), else 0;
                     // 4: coefficient table (rows = orders, row stride rs = 2L+1) in term order kk
                     // 5: an operand of a COMPLEX product as one real GEMM (ozgemm CM 1): z(r, k)
                     //    = src complex element r * rs + k * ks (complex strides), K doubled:
                     //    ra = 0 (A side): A'(r, 2k + e) = e ? -Im z : Re z
                     //    ra = 1 (B side, rows 2j + c): B'(2j + c, 2k + e) = (Re, Im; Im, -Re)[c][e]
                     //    ka = 1: conjugate z first
                     // 7: element-pair rows of the PAIR-MAJOR digit cache (the INT8 synthesis,
                     //    dsynth_kernel): row r -> M tile mt = r / 128, pair p = mt / 8, t = 128
                     //    (mt % 8) + r % 128, (I, J) = pair_of_imajor(p), i = t % 32, j = t / 32;
                     //    K < kp / 2: P_(K+1)(32 I + i, 32 J + j), K >= kp / 2: the mirror
                     //    P_(K-kp/2+1)(32 J + j, 32 I + i) (tiled slabs: sbatch = slab elements,
                     //    nt, l = L, tp2 = n)
                     // 8: node coefficient rows for element-pair operands (ozgemm pair mode):
                     //    row 2x + m, K < kp / 2: c_x(+-(K + 1)), K >= kp / 2: c_x(-+(K - kp/2 + 1))
                     //    (+ for m = 0 in the first half); src = r x rs table, c_k at column l + k
                     // 6: element rows of the stacked cache (the basis synthesis GEMM): row
                     //    e = i + j n (rv = n^2, tp2 = n), K term kk < L: P_(kk+1)(i, j), L <= kk < 2L:
                     //    P_(kk-L+1)(j, i); one batch block (nb = 1, rp = padded n^2)
    int nt = 0;      // tiles per side of a tiled slab
    int l = 0, tp2 = 0;  // modes 3 / 4: L and the padded term count (64 or 128)
    int64_t rmb = 0;     // slicing from ready row maxima: slot of row (bt, r) = bt * rmb + r (0: bt * rp + r)
};


// Output addressing: row m -> (batch block bm = m / mp, i = m % mp), valid when i < mv, n < nv.
//   CM 0: C[bm * sC + i + n * ldc]                       (real, column-major)
//   CM 1: C[bm * sC + (i + (n >> 1) * ldc) * 2 + (n & 1)]  (complex merge of column pairs)
//   CM 2: power products of the orthogonal-F sweep -> base-254 digits of Z for the combine GEMM
//         plus Gram partials (rows m = i * tp2 + kk: signal row i, term kk; columns 2j + comp)
//   CM 3: the combine GEMM Y = C Z (rows = flat positions p, columns = orders) + c_0 X, the
//         optional store of Y and the per-order MSE loss partials.
struct OzOut {
    double* c;
    int64_t ldc, sc;
    int mv, mp, nv;
    // CM 2 / CM 3 extras
    const double* x = nullptr;   // X, flat 2 n b doubles
    const double* xc = nullptr;  // clean signals (CM 3) / Xc (CM 2 Gram partials)
    const double* zl = nullptr;  // unused (kept for layout stability)
    const int* epos = nullptr;   // CM 2: exponent per signal column j: |Z_k[i, j]| < 2^e
    int8_t* zd = nullptr;        // CM 2: digits, A operand layout of the combine GEMM
    double* part = nullptr;      // CM 2: [cta][2][128][3] Gram partials; CM 3: [cta][2][4][32] loss
    const double* c0 = nullptr;  // CM 3: c_0 of order a at c0[a * c0s]
    int64_t c0s = 1;
    int64_t count = 0;           // 2 n b
    int n = 0, tp2 = 0, kbz = 0; // signal length, padded terms (64 | 128), K blocks of the combine
    int l = 0;                   // CM 2: L (row kk = 2L-1 holds Z_-L)
    // CM 0 / 1: the same tile also stored at these bases (peer GPUs' buffers mapped over NVLink:
    // the all-gather of a row-sharded output fused into the GEMM epilogue). Offsets as for c.
    double* peers[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    int npeers = 0;
    // CM 0, skinny (nv <= 32) node operators over element rows m = i + j rn (rn % 128 == 0): the
    // grid is a multiple of rn / 128 so each CTA stays in one row block; adds dg[col] on the diagonal
    // (i == j) and leaves max_j |C[i + j rn, col]| in rmax[col * rnp + i] (atomicMax on the bits of
    // a non-negative double; zeroed by the caller) -- the row max the product GEMM's slicing needs.
    unsigned long long* rmax = nullptr;
    const double* dg = nullptr;
    int rn = 0, rnp = 0;
    int max_ctas = 0;  // > 0: cap the persistent grid (leave SMs to a concurrent kernel)
    // CM 1 fused reduce-scatter (pair shards): complex output column j goes to owner h = j / scw
    // instead of c: dest[h] + bm * ssc + (i + (j - h scw) * sld) * 2 -- each owner's receive slot for
    // this rank, local or a peer GPU's buffer mapped over NVLink (CUDA IPC). scw = 0: off.
    double* dest[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    int scw = 0;
    int64_t ssc = 0, sld = 0;
    // CM 1: the diagonal term of a series whose synthesis left out c_0 I (A = Q - c_0 I, so the
    // slicing error follows the off-diagonal entries): C[bm] += dgc[bm * dgs] * dx[same offset as C
    // within a block] (dx complex, laid out as C with the same ldc). dx = nullptr: off.
    const double* dx = nullptr;
    const double* dgc = nullptr;
    int64_t dgs = 0;
    // CM 0 node operators over ELEMENT-PAIR rows (A = the pair-major slices of OzView mode 7, B =
    // mode 8 coefficient rows): pair_nt > 0 = tiles per side. Output column 2x + m is node x's
    // operator at element e (m = 0) or its mirror e' (m = 1), stored at c + x * ldc + column-major
    // (pair_n x pair_n); dg[x] added on the diagonal; rmax[x * rnp + row] = the row maxima (zeroed
    // by the caller). Each CTA takes the 8 M tiles of a tile pair in a row.
    int pair_nt = 0, pair_n = 0;
    // CM 1: N-band raster (set by the launcher). The unit order walks all M tiles over band 0's N
    // groups, then band 1's, ...: a B operand larger than L2 (config 4: 151 MB of X digits) stays
    // resident one band at a time instead of being re-streamed from HBM by every wave of M tiles.
    int nband = 1;
    // CM 1 fused MSE + dL/da (the packed step, DESIGN 3.7): A = [Q_a blocks; dQ_a blocks] (2 n_alpha
    // blocks of mp rows, an even number of M tiles); each CTA takes M tile mt and then mt + mtiles / 2
    // (the dQ rows of the same Q rows) with the same N tile, so the thread that stored Y[i, j] meets
    // dY[i, j] one unit later: the Y tile is stored and sum |Y - Xc|^2 accumulated, the dY tile is NOT
    // stored and sum Re conj(Y - Xc) dY accumulated (Y read back from c, block bm - n_alpha). Warp
    // sums per Y tile (mt < mtiles / 2, nt) land in lpart[((mt * ntiles + nt) * 16 + ew) * 2 + {0, 1}]
    // (fixed order: the finish kernel's sums are deterministic). lxc: Xc, laid out as C in a block.
    double* lpart = nullptr;
    const double* lxc = nullptr;
};

constexpr int kOzTileA = 128;  // A operand row tile (output rows per CTA)
constexpr int kOzTileNarrow = 32;  // B row tile of the skinny node-operator GEMM
constexpr int kOzTileB = 64;   // B operand row tile (output columns per CTA)
constexpr int kOzK = 64;       // K padding granule

int oz_slices_default();
// INT8 tensor-core synthesis (ozgemm.cu dsynth_kernel): operator rows x < ac of
// Q_x = c_x0 I + sum_k c_xk P_k + c_x(-k) P_k^T for the tile pairs [p0, p1) (p1 < 0: all) from the
// pair-major element-row digit cache (launch_dsynth_build) and the coefficient digits
// (launch_dsynth_coefs); out + x out_stride: n x n column-major, rowmax + x mp: row maxima.
size_t dsynth_cache_rows(int n);
int dsynth_slices();
int dsynth_kp(int l);  // K of the digit cache: 2 x pad64(L)
size_t dsynth_coef_bytes(int kp);
cudaError_t launch_dsynth_build(const double* slabs, int n, int l, int kp, int8_t* digits, int* exps,
                                unsigned long long* rowmax_tmp, cudaStream_t stream, int slices = 0);
size_t dsynth_cache_rows(int n);  // element-pair rows (128-row tiles, 8 per tile pair)
cudaError_t launch_dsynth_coefs(const double* coef, int coef_ld, int l_used, int ac, int kp, int8_t* bsl,
                                cudaStream_t stream);
cudaError_t launch_dsynth(const int8_t* digits, const int* exps, const int8_t* bsl, int kp, int n, int p0, int p1,
                          const double* coef, int coef_ld, int l_used, int ac, double* out, int64_t out_stride,
                          unsigned long long* rowmax, int64_t mp, int max_ctas, cudaStream_t stream, int nodiag = 0);
// Slice a viewed operand into dst (slices * nb * rp * kp bytes) + exps (nb * rp ints);
// rowmax: nb * rp scratch words. tr = kOzTileA for an A operand, kOzTileB for a B operand.
cudaError_t launch_oz_slice(const OzView& v, int slices, int tr, int8_t* dst, int* exps, unsigned long long* rowmax,
                            cudaStream_t stream);
// C = A B^T over sliced operands; cm 0: C[bm*sc + i + n*ldc], cm 1: complex merge of column
// pairs C[bm*sc + (i + (n>>1)*ldc)*2 + (n&1)], with m = bm * mp + i (i < mv), n < nv.
cudaError_t launch_ozgemm_narrow(int slices, const int8_t* a, const int* ea, int mrows, const int8_t* b,
                                 const int* eb, int nrows, int kp, const OzOut& out, cudaStream_t stream);
cudaError_t launch_oz_slice_ready(const OzView& v, int slices, int tr, int8_t* dst, int* exps,
                                  const unsigned long long* rowmax, cudaStream_t stream);
cudaError_t launch_ozgemm_ex(int slices, int cm, const int8_t* a, const int* ea, int mrows, const int8_t* b,
                             const int* eb, int nrows, int kp, const OzOut& out, cudaStream_t stream);
int oz_bk(int slices);  // bytes of K per stage / per digit block of the sliced layout
int oz_zdigits();       // digits of Z written by the CM 2 epilogue (the combine GEMM's digit count)
cudaError_t launch_ozgemm(int slices, int cm, const int8_t* a, const int* ea, int mrows, const int8_t* b,
                          const int* eb, int nrows, int kp, double* c, int64_t ldc, int64_t sc, int mv, int mp, int nv,
                          cudaStream_t stream, double* const* peers = nullptr, int npeers = 0, int max_ctas = 0);

}  // namespace fgb
