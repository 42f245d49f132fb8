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
                     // 2: the same slab read transposed, element (r, k) = P(k, r)
    int nt = 0;      // tiles per side of a tiled slab
};


constexpr int kOzTileA = 128;  // A operand row tile (output rows per CTA)
constexpr int kOzTileB = 64;   // B operand row tile (output columns per CTA)
constexpr int kOzK = 64;       // K padding granule

int oz_slices_default();
// Slice a viewed operand into dst (slices * nb * rp * kp bytes) + exps (nb * rp ints);
// rowmax: nb * rp scratch words. tr = kOzTileA for an A operand, kOzTileB for a B operand.
cudaError_t launch_oz_slice(const OzView& v, int slices, int tr, int8_t* dst, int* exps, unsigned long long* rowmax,
                            cudaStream_t stream);
// C = A B^T over sliced operands; cm 0: C[bm*sc + i + n*ldc], cm 1: complex merge of column
// pairs C[bm*sc + (i + (n>>1)*ldc)*2 + (n&1)], with m = bm * mp + i (i < mv), n < nv.
cudaError_t launch_ozgemm(int slices, int cm, const int8_t* a, const int* ea, int mrows, const int8_t* b,
                          const int* eb, int nrows, int kp, double* c, int64_t ldc, int64_t sc, int mv, int mp, int nv,
                          cudaStream_t stream);

}  // namespace fgb
