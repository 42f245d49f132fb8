/*
 * fgfrft_b200.h -- C ABI of the B200-native FGFRFT hot path (libfgfrft_b200.so).
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++/torch types. The C++
 * drop-in header include/fgfrft/transform.hpp (same names and semantics as the reference
 * header proj/include/fgfrft/transform.hpp) forwards every call here; a ctypes / cgo /
 * JNI binding would bind exactly these symbols.
 *
 * Matrix convention (identical to Eigen::MatrixXcd, which the reference uses):
 *   column-major, interleaved (re, im) doubles; element (i, j) of an n x n matrix is at
 *   doubles [2*(i + j*n)] and [2*(i + j*n) + 1]. Signal blocks X are n x b, column-major.
 *   complex64 caches take/return the same complex128 host buffers; storage and arithmetic
 *   on the device are complex64 (fgfrft_dtype FGFRFT_C64). For a real F (imaginary part exactly
 *   zero) a C64 cache stores the powers as real doubles -- the same 8 bytes per element -- and
 *   computes in FP64; its *_dev entry points still take and return complex64 device signals.
 *
 * Series layout (identical to SincCoeffs, proj/include/fgfrft/sinc.hpp:40-48): arrays of
 *   2L+1 doubles where entry [n + L] holds term n, n = -L..L.
 *
 * Errors: every function returns an fgfrft_status; no C++ exception crosses this boundary.
 * The message of the last failure on the calling thread is fgfrft_last_error().
 * Mapping to the reference exception taxonomy (proj/include/fgfrft/errors.hpp:36-62):
 *   FGFRFT_PARAMETER -> parameter_error, FGFRFT_SHAPE -> shape_error,
 *   FGFRFT_CAPACITY -> capacity_error, FGFRFT_NUMERICAL / FGFRFT_CUDA / FGFRFT_NCCL ->
 *   numerical_error, FGFRFT_OPTIMIZER -> optimizer_error (a numerical_error), FGFRFT_IO ->
 *   io_error, FGFRFT_PARSE -> parse_error.
 *
 * Threading: calls on one handle are serialised by the handle; distinct handles may be
 * used concurrently. Every call is synchronous with respect to host buffers. Calls taking
 * device pointers (the *_dev variants) enqueue on the handle's stream and return without
 * synchronising; fgfrft_cache_set_stream selects that stream.
 */
#ifndef FGFRFT_B200_H
#define FGFRFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fgfrft_status {
    FGFRFT_OK = 0,
    FGFRFT_PARAMETER = 1,
    FGFRFT_SHAPE = 2,
    FGFRFT_CAPACITY = 3,
    FGFRFT_NUMERICAL = 4,
    FGFRFT_CUDA = 5,
    FGFRFT_NCCL = 6,
    FGFRFT_OPTIMIZER = 7, /* non-finite loss / gradient in a learner (optimizer_error) */
    FGFRFT_IO = 8,        /* file cannot be opened / written (io_error) */
    FGFRFT_PARSE = 9      /* malformed or truncated file (parse_error) */
} fgfrft_status;

typedef enum fgfrft_dtype { FGFRFT_C128 = 0, FGFRFT_C64 = 1 } fgfrft_dtype;

typedef enum fgfrft_which { FGFRFT_Q = 0, FGFRFT_DQ = 1 } fgfrft_which;

/*
 * GEMM engine of a handle (fgfrft_cache_set_engine). DMMA: FP64 tensor cores (mma.sync f64),
 * every order synthesised then multiplied. INT8: for real F, order sweeps run through the
 * power products F^k X computed by one Ozaki-scheme GEMM on the INT8 tensor cores
 * (tcgen05 kind::i8; ~3e-13 relative, see fgfrft_dgemm_int8_dev). AUTO (default, or the
 * FGFRFT_ENGINE=dmma|int8 environment variable): INT8 power products when 2 n_alpha >= L.
 */
typedef enum fgfrft_engine {
    FGFRFT_ENGINE_AUTO = 0,
    FGFRFT_ENGINE_DMMA = 1,
    FGFRFT_ENGINE_INT8 = 2,
    /* INT8, and for an orthogonal F with 32 <= L <= 64 also the per-order combination Y = C Z on
     * the INT8 tensor cores (Z written as digits by the power-product GEMM). Experimental. */
    FGFRFT_ENGINE_INT8_COMBINE = 3
} fgfrft_engine;

/* Default budget of transform.hpp:17 (4 GiB). */
#define FGFRFT_DEFAULT_MEMORY_BUDGET (4ULL << 30)

typedef struct fgfrft_cache fgfrft_cache;
typedef struct fgfrft_spectrum fgfrft_spectrum; /* spectral form of F, see below */

/* ---- library ----------------------------------------------------------------------- */

/* Message of the last failing call on this thread ("" if none). */
const char* fgfrft_last_error(void);

/* Version string of the library ("0.1.0-b200"). */
const char* fgfrft_version(void);

/* Number of kernel launches this process has issued through the library (monotone). */
uint64_t fgfrft_launch_count(void);

/*
 * Per-kernel-class device timing (CUDA events on the launching stream), for benchmarks:
 * classes 0 synthesis, 1 DMMA GEMM, 2 power dots, 3 elementwise, 4 INT8 tensor-core GEMM,
 * 5 operand slicing, 6 series combine, 7 node operators (order-sweep node route). fgfrft_profile_read waits for the recorded
 * events, writes total ms and launch counts per class (arrays of 8) and optionally resets.
 */
int fgfrft_profile_enable(int on);
int fgfrft_profile_read(double* ms, int64_t* counts, int reset);
/* The recorded launches in order (before a reset): class, start and end in ms relative to the first
 * record's start (CUDA events on the launching streams); up to cap records, *count = recorded. */
int fgfrft_profile_trace(int* cls, double* t0, double* t1, int cap, int* count);

/* sinc.hpp:50-63. c, dc: 2l+1 doubles each (either may be NULL). l < 1 -> PARAMETER. */
int fgfrft_sinc_coeffs(double alpha, int l, double* c, double* dc);

/* FNV-1a-64 over nbytes (rng.hpp:59-67), the cache fingerprint (gft.hpp:46-48). */
uint64_t fgfrft_fnv1a64(const void* data, size_t nbytes);

/* ---- power cache: replaces PowerCache (transform.hpp:41-80) ------------------------- */

/*
 * Build P_k = F^k, k = 1..l, on device `device` (transform.hpp:43-59): budget check
 * l*n*n*elem > memory_budget -> CAPACITY (elem = 16 for C128, 8 for C64), FNV-1a
 * fingerprint of f, P_1 = F, P_k = F P_{k-1} on FP64 tensor cores (DMMA).
 * f: n x n host matrix (see convention). l < 1 or n < 1 -> PARAMETER.
 */
int fgfrft_cache_create(const double* f, int64_t n, int l, uint64_t memory_budget, int dtype,
                        int device, fgfrft_cache** out);

/* Same, but from host-built powers (l slabs, slab k-1 = F^k) -- no recursion on device. */
int fgfrft_cache_create_from_powers(const double* powers, const double* f, int64_t n, int l,
                                    uint64_t memory_budget, int dtype, int device,
                                    fgfrft_cache** out);

int fgfrft_cache_destroy(fgfrft_cache* cache);

/* n, l, fingerprint, dtype, device (any pointer may be NULL). */
int fgfrft_cache_info(const fgfrft_cache* cache, int64_t* n, int* l, uint64_t* fingerprint,
                      int* dtype, int* device);

/* 1 if F's imaginary part is exactly zero: the cache is stored as real doubles and the real-F
 * kernels run (half the bytes and flops; results equal the complex path's up to rounding).
 * Set FGFRFT_NO_REAL=1 in the environment to force the complex kernels. */
int fgfrft_cache_is_real(const fgfrft_cache* cache, int* real);
/* Route taken by the last fgfrft_mse_step* on this handle: 0 synthesis (one GEMM pair per order),
 * 1 power products (2L products F^k X), 2 node interpolation (nodes = its r node operators),
 * 3 packed step (Q, dQ/da from the packed 40-bit slabs, then one INT8 Ozaki GEMM), 4 the same step
 * with Q, dQ/da synthesised on the INT8 tensor cores from the element-row digit cache; -1 before
 * the first step. For benchmarks and diagnostics. */
int fgfrft_cache_route_info(const fgfrft_cache* cache, int* route, int* nodes);

/* transform.hpp:131-134: copy F^k (1 <= k <= l, else PARAMETER) to host (n x n). */
int fgfrft_cache_power(fgfrft_cache* cache, int k, double* out);

/* transform.hpp:136-139: NUMERICAL if fnv1a64(f) != stored fingerprint. */
int fgfrft_cache_verify(const fgfrft_cache* cache, const double* f);

/* Stream for subsequent calls on this handle (cudaStream_t as void*; NULL = the CUDA default
 * stream, as everywhere in CUDA). A new handle uses its own non-blocking stream. */
int fgfrft_cache_set_stream(fgfrft_cache* cache, void* stream);

/* Device pointer to slab k-1 (= F^k) and the device memory held by the handle. */
int fgfrft_cache_set_engine(fgfrft_cache* cache, int engine);
/* ||F^T F - I||_F / sqrt(n) measured on the device when a real cache is built (gft.hpp:39-44
 * normalisation); -1 for complex caches. <= 1e-12 enables the Gram form of the power-product
 * MSE step (s_k from <X, F^d X>). */
int fgfrft_cache_orthogonality(const fgfrft_cache* cache, double* residual);
/* Build lazily-built device structures now (the INT8 digit slices of the stacked cache for the
 * power-product route); a no-op for handles that never use them. Synchronises. */
int fgfrft_cache_prepare(fgfrft_cache* cache);

// Order window (an extension, no reference counterpart): declare the orders the caller will step
// with. Builds r exact FP64 node operators Q(x_j) - c_0(x_j) I at the Chebyshev nodes of [lo, hi]
// (r ~ 9 + 5 (hi - lo); r n^2 8 bytes, counted against the memory budget), after which the one- /
// two-order step and apply routes synthesise Q(a), dQ/da of orders inside [lo, hi] from them --
// r slabs instead of the L powers (the coefficients are interpolated to 4e-15 of the largest;
// orders outside the window take the packed route). hi <= lo clears it. Real F, n >= 512 only.
int fgfrft_cache_set_order_window(fgfrft_cache* cache, double lo, double hi);
int fgfrft_cache_order_window(const fgfrft_cache* cache, double* lo, double* hi, int* nodes);
int fgfrft_cache_device_slab(fgfrft_cache* cache, int k, void** dptr);
int fgfrft_cache_device_bytes(const fgfrft_cache* cache, uint64_t* bytes);

/* ---- series synthesis: replaces fgfrft_matrix / fgfrft_grad (transform.hpp:111-136) -- */

/*
 * For each of n_alpha orders: Q = c_0 I + sum_{k=1..L'} (c_k F^k + c_{-k} (F^k)^H) with
 * c = sinc coefficients (which = FGFRFT_Q) or their alpha-derivatives (FGFRFT_DQ).
 * L' = truncation (0 -> cache l; L' > l or < 0 -> PARAMETER; DQ always uses the full l).
 * out: n_alpha consecutive n x n host matrices.
 */
int fgfrft_synthesize(fgfrft_cache* cache, const double* alphas, int n_alpha, int truncation,
                      int which, double* out);

/* Device variant: out_dev = n_alpha consecutive n x n device matrices of the cache dtype. */
int fgfrft_synthesize_dev(fgfrft_cache* cache, const double* alphas, int n_alpha,
                          int truncation, int which, void* out_dev);

/* ---- apply: replaces apply_forward / apply_inverse (transform.hpp:138-148) ----------- */

/*
 * Y_a = Q(alpha_a) X (inverse = 0) or Q(alpha_a)^H X (inverse = 1) for n_alpha orders,
 * Q synthesised on the device and consumed by the DMMA complex GEMM without a host
 * round trip. x: n x b host; y: n_alpha consecutive n x b host blocks.
 */
int fgfrft_apply(fgfrft_cache* cache, const double* alphas, int n_alpha, int truncation,
                 int inverse, const double* x, int64_t b, double* y);
int fgfrft_apply_dev(fgfrft_cache* cache, const double* alphas, int n_alpha, int truncation,
                     int inverse, const void* x_dev, int64_t b, void* y_dev);

/*
 * Plain apply of a materialised operator (FracOperator.q) -- apply_forward(op, X) exactly:
 * Y = Q X (inverse = 0) or Q^H X (inverse = 1), Q: n x n host, X: n x b host, complex128.
 * Runs the same DMMA GEMM on device `device`.
 */
int fgfrft_apply_matrix(const double* q, int64_t n, int inverse, const double* x, int64_t b,
                        double* y, int device);

/* ---- order gradient: dL/dalpha = sum_k c'_k(alpha) Re<G, F^k X> (learn.hpp:88-92) ---- */

/*
 * For each order a: s_{a,k} = Re<G_a, F^k X> for k = -L..L (written to s, n_alpha x (2L+1),
 * may be NULL) and dlda[a] = sum_k c'_k(alpha_a) s_{a,k}. g: n_alpha consecutive n x b
 * cotangents (dL/dconj(Y) convention of learn.hpp:92: L = ||R||^2 -> G = 2R / norm).
 */
int fgfrft_dlda(fgfrft_cache* cache, const double* alphas, int n_alpha, const double* g,
                const double* x, int64_t b, double* s, double* dlda);
int fgfrft_dlda_dev(fgfrft_cache* cache, const double* alphas, int n_alpha, const void* g_dev,
                    const void* x_dev, int64_t b, double* s, double* dlda);

/*
 * MSE denoising step over an order sweep (the BASELINE config-2 workload): for each order a,
 * Y_a = Q(alpha_a) X, loss_a = ||Y_a - Xc||_F^2 / (n b), G_a = 2 (Y_a - Xc) / (n b) and
 * dlda_a = dloss_a/dalpha = sum_k c'_k(alpha_a) Re<G_a, F^k X>.
 * Host variant: x, xc host (pinned for full speed), y host or NULL; loss, dlda host arrays of
 * n_alpha; synchronous. Device variant: all pointers device, enqueued on the handle stream.
 */
int fgfrft_mse_step(fgfrft_cache* cache, const double* alphas, int n_alpha, const double* x,
                    const double* xc, int64_t b, double* y, double* loss, double* dlda);
int fgfrft_mse_step_dev(fgfrft_cache* cache, const double* alphas, int n_alpha,
                        const void* x_dev, const void* xc_dev, int64_t b, void* y_dev,
                        void* loss_dev, void* dlda_dev);

/* ---- row-slab shards for multi-GPU -------------------------------------
 *
 * A shard owns output rows R = [row_begin, row_end) (row_begin % 32 == 0; row_end % 32 == 0
 * or row_end == n) and stores the row panels P_k[R,:] and column panels P_k[:,R], k = 1..l
 * (the rows of F^k and of F^{-k}), built on device from the replicated F. Everything below is
 * local to the shard; the caller combines ranks with one all-reduce of the 2l+1 partials (and
 * the loss) and one gather of the rows. Budget: 2*l*rows*n*16 bytes. The handle type is
 * fgfrft_cache; the non-shard entry points reject it (and vice versa).
 * Row blocks are column-major with leading dimension rows = row_end - row_begin.
 */
int fgfrft_shard_create(const double* f, int64_t n, int l, int64_t row_begin, int64_t row_end,
                        uint64_t memory_budget, int device, fgfrft_cache** out);
int fgfrft_shard_destroy(fgfrft_cache* shard);
int fgfrft_shard_info(const fgfrft_cache* shard, int64_t* n, int* l, int64_t* row_begin,
                      int64_t* row_end, uint64_t* fingerprint);
int fgfrft_shard_set_stream(fgfrft_cache* shard, void* stream);
/* Q(alpha_a)[R,:] (or dQ) for n_alpha orders: out_dev = n_alpha blocks of rows x n. */
int fgfrft_shard_synthesize_dev(fgfrft_cache* shard, const double* alphas, int n_alpha, int which,
                                void* out_dev);
/* Y[R,:] = Q(alpha_a)[R,:] X; x_dev n x b (replicated), y_dev n_alpha blocks of rows x b. */
int fgfrft_shard_apply_dev(fgfrft_cache* shard, const double* alphas, int n_alpha,
                           const void* x_dev, int64_t b, void* y_dev);
/* Per order: loss_partial[a] = ||Y[R,:] - Xc[R,:]||^2 (unnormalised), s_partial[a][k+l] =
 * Re<G[R,:], (F^k X)[R,:]> with G = 2 (Y - Xc) / (n b). xc_rows_dev: rows x b. y_rows_dev may be
 * NULL. All outputs are device arrays. Sum both over ranks; then loss = sum / (n b) and
 * dL/dalpha = sum_k c'_k s_k. */
int fgfrft_shard_mse_partial_dev(fgfrft_cache* shard, const double* alphas, int n_alpha,
                                 const void* x_dev, const void* xc_rows_dev, int64_t b,
                                 void* y_rows_dev, void* loss_partial_dev, void* s_partial_dev);
/* Fused all-gather of the apply (north star: "the final row gather"): rows [r0, r1) of
 * Y_a = F^alpha_a X are written into y_full_dev (n_alpha blocks of n x b, column-major, the FULL
 * result) AND, at the same offsets, into each of the n_peers peer buffers peer_y_full[q] -- the
 * other ranks' y_full buffers mapped into this process (fgfrft_ipc_open) -- by the INT8 GEMM's
 * epilogue itself (NVLink P2P stores interleaved with the tiles), or by a P2P push kernel after the
 * DMMA GEMM. After every rank's call has completed (stream sync + a host barrier), every y_full
 * holds all rows. n_peers <= 7. */
int fgfrft_shard_apply_gather_dev(fgfrft_cache* shard, const double* alphas, int n_alpha,
                                  const void* x_dev, int64_t b, void* y_full_dev,
                                  void* const* peer_y_full, int n_peers);
/* CUDA IPC for the peer mappings: handle (64 bytes) and the offset of dev_ptr inside its
 * allocation; open maps a peer's allocation (base) on `device`; close unmaps it. */
int fgfrft_ipc_get(const void* dev_ptr, void* handle_out, uint64_t* offset_out);
int fgfrft_ipc_open(const void* handle, int device, void** base_out);
int fgfrft_ipc_close(void* base);
/* Same, returning dlda_partial[a] = sum_k c'_k(alpha_a) s_partial[a][k] directly (n_alpha doubles
 * to all-reduce instead of n_alpha (2L+1)); one or two orders synthesise dQ/dalpha rows in the
 * same pass over the panels as Q and take Re<M[R,:], dQ[R,:]>, no second pass. */
int fgfrft_shard_mse_dlda_partial_dev(fgfrft_cache* shard, const double* alphas, int n_alpha,
                                      const void* x_dev, const void* xc_rows_dev, int64_t b,
                                      void* y_rows_dev, void* loss_partial_dev, void* dlda_partial_dev);

/* ---- Multi-GPU: NCCL communicator + pair shards of the packed cache ----------------------
 *
 * Replaces the single-GPU PowerCache (transform.hpp:43-59) + MSE step for caches sharded over
 * the GPUs of one node, without PyTorch: the library owns the NCCL communicator (libnccl.so.2,
 * loaded at first use). Bootstrap like NCCL itself: rank 0 calls fgfrft_comm_unique_id and the
 * launcher hands the 128 bytes to every rank (MPI, a TCP store, torch.distributed, ...); or one
 * process drives all devices with fgfrft_comm_create_all (ncclCommInitAll).
 *
 * A pair shard owns the tile pairs {(I,J),(J,I)}, I <= J, with I in its contiguous band (about
 * 1/G of the pairs; fgfrft_pshard_plan gives the bands), stores only their packed powers (5 B
 * per element, built from its row / column panels -- F is broadcast from rank 0, the only
 * collective of the build), synthesises Q, dQ/da on its tiles and multiplies them with X locally.
 * Per MSE step: one reduce-scatter of [Y; dY] by signal-column chunks and one all-reduce of 2A
 * doubles. Real F (graph GFTs) only; a complex F uses the row shards above.
 */
#define FGFRFT_COMM_ID_BYTES 128
typedef struct fgfrft_comm fgfrft_comm;
int fgfrft_comm_unique_id(void* id_out /* FGFRFT_COMM_ID_BYTES */);
int fgfrft_comm_create(const void* id, int world, int rank, int device, fgfrft_comm** out);
int fgfrft_comm_create_all(int ndev, const int* devices, fgfrft_comm** out /* ndev handles */);
int fgfrft_comm_destroy(fgfrft_comm* comm);
int fgfrft_comm_info(const fgfrft_comm* comm, int* world, int* rank, int* device);

/* Tile-row band boundaries (world + 1 ints, in 32-row tiles) of the pair shards of an n x n F. */
int fgfrft_pshard_plan(int64_t n, int world, int* tile_rows);
/* f: n x n complex128 column-major on every rank, or NULL on ranks != 0 (broadcast from rank 0). */
int fgfrft_pshard_create(const double* f, int64_t n, int l, uint64_t memory_budget, fgfrft_comm* comm,
                         fgfrft_cache** out);
/* A shard of rank `rank` of `world` with no communicator (partials only: tests, custom reductions). */
int fgfrft_pshard_create_local(const double* f, int64_t n, int l, uint64_t memory_budget, int world, int rank,
                               int device, fgfrft_cache** out);
int fgfrft_pshard_destroy(fgfrft_cache* shard);
int fgfrft_pshard_info(const fgfrft_cache* shard, int* world, int* rank, int64_t* pair_begin, int64_t* pair_end,
                       int64_t* row_begin, int64_t* row_end, uint64_t* device_bytes);
int fgfrft_pshard_set_stream(fgfrft_cache* shard, void* stream);
/* This rank's partial products (sum over ranks = the full result): with_dq 1 -> 2 n_alpha blocks
 * [Y_g(a..); dY_g(a..)], 0 -> n_alpha blocks Y_g(a..), each n x b complex (stride 2 n b doubles). */
int fgfrft_pshard_partial_dev(fgfrft_cache* shard, const double* alphas, int n_alpha, int with_dq,
                              const void* x_dev, int64_t b, void* out_dev);
/* The same partial products scattered by signal-column chunk straight from the GEMM epilogue (the
 * data path of the fused reduce-scatter the MSE step runs over NVLink): dest[h] = this rank's
 * receive slot in owner h's buffer, rows blocks of n x cb complex (cb = ceil(b / ndest), ndest <= 8);
 * summing owner h's slots over the source ranks gives columns [h cb, (h+1) cb) of the result. */
int fgfrft_pshard_partial_scatter_dev(fgfrft_cache* shard, const double* alphas, int n_alpha, int with_dq,
                                      const void* x_dev, int64_t b, void* const* dest, int ndest);
/* MSE step (one or two orders) over the communicator; full X, Xc on every rank; loss and
 * dL/dalpha of every order on every rank. */
int fgfrft_pshard_mse_step_dev(fgfrft_cache* shard, const double* alphas, int n_alpha, const void* x_dev,
                               const void* xc_dev, int64_t b, void* loss_dev, void* dlda_dev);
int fgfrft_pshard_mse_step(fgfrft_cache* shard, const double* alphas, int n_alpha, const double* x,
                           const double* xc, int64_t b, double* loss, double* dlda);
/* Y = F^alpha X (inverse: the conjugate transpose) for 1, 2 or 4 orders, the full Y on every rank. */
int fgfrft_pshard_apply_dev(fgfrft_cache* shard, const double* alphas, int n_alpha, int inverse,
                            const void* x_dev, int64_t b, void* y_dev);

/* ---- FP64-accurate GEMM on the INT8 tensor cores (Ozaki scheme) -------------------------
 *
 * C = op(A) op(B) for real column-major device matrices (op(A) m x k, op(B) k x n, C m x n;
 * op(X) = X^T when trans* != 0, as in BLAS dgemm), computed with
 * tcgen05.mma kind::i8: A's rows and B's columns are scaled by powers of two and cut into
 * `slices` balanced base-254 digits (6, 7 or 8; 0 = default 6); digit products of weight
 * >= 254^-(S+1) accumulate exactly in int32 TMEM and are combined in FP64. Error ~ sqrt(k)
 * 254^-S relative to (row max of A) x (column max of B): 6 digits (21 int8 products) ~3e-13 on
 * the BASELINE operands, 7 digits (28 products) ~1e-15.
 * k <= 16384. Enqueued on `stream` (NULL = default stream); scratch is allocated per call.
 * This is the engine behind the library's real-F GEMMs (fgfrft_set_gemm_engine).
 */
/* Default digit count of the library's INT8 engine (6). */
int fgfrft_int8_digits(void);
/* Digits per operand of the packed step route's product GEMM [Y; dY] = [Q; dQ] X (routes 3 / 4):
 * 5 by default (Q carries the cache's ~2^-40 quantisation), FGFRFT_STEP_SLICES=6 for 6. */
int fgfrft_step_int8_digits(void);
/* Complex128 GEMM on the same engine: C (m x n, column-major ldc) = op(A) op(B), trans 0 = N,
 * 1 = T, 2 = C (conjugate transpose); interleaved (re, im) doubles. Computed as ONE real Ozaki
 * GEMM with K doubled (A' = [Re, -Im], B' = [[Re, Im], [Im, -Re]] per element, the epilogue merges
 * column pairs into (Re C, Im C)): 8 m n k FP64-equivalent flops. k <= 8192. */
int fgfrft_zgemm_int8_dev(int transa, int transb, int64_t m, int64_t n, int64_t k, const double* a,
                          int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc,
                          void* stream);
int fgfrft_dgemm_int8_dev(int transa, int transb, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda,
                          const double* b, int64_t ldb, double* c, int64_t ldc, int slices,
                          void* stream);

/* ---- GPU-resident denoising learner (learn.hpp:291-516, adam.hpp) -------------------------
 *
 * The paper's denoising workload on the device (fast backend; real or complex F): every evaluation
 * synthesises Q(alpha) and dQ/dalpha from the cache in one pass (alpha lives on the device; its
 * sinc coefficients are evaluated there, ~1 ulp from glibc) and forms, with five n x n x C GEMMs
 * (INT8 engine or DMMA), the quantities of the reference's fast engine:
 *   u = Q y, w = Q^H (h o u), loss = |w - x|^2, grad_h = 2 rowsum(Q r o u),
 *   grad_alpha = 2 <r, dQ^H/dalpha (h o u)> + 2 <Q r, h o dQ/dalpha y>,  r = w - x.
 * y, x_ref, reconstruction: n x channels real, column-major (host). fit runs Adam (lr, beta
 * 0.9 / 0.999, eps 1e-8) over [alpha, h] from [init_alpha, 1..1] for `epochs` steps, evaluating
 * once more at the end (trajectories have epochs + 1 entries) and tracking the best loss, all on
 * the device; a non-finite loss / gradient inside the loop -> FGFRFT_OPTIMIZER naming the epoch.
 */
typedef struct fgfrft_denoise fgfrft_denoise;
int fgfrft_denoise_create(fgfrft_cache* cache, const double* y, const double* x_ref, int64_t channels,
                          fgfrft_denoise** out);
/* Same with the loss on the real part of the reconstruction (loss_on_real, learn.hpp:389-403;
 * only differs from the plain form for a complex F). A complex F runs the same five products as
 * complex GEMMs. */
int fgfrft_denoise_create_ex(fgfrft_cache* cache, const double* y, const double* x_ref, int64_t channels,
                             int loss_on_real, fgfrft_denoise** out);
int fgfrft_denoise_destroy(fgfrft_denoise* problem);
int fgfrft_denoise_eval(fgfrft_denoise* problem, double alpha, const double* h, double* loss,
                        double* grad_alpha, double* grad_h);
int fgfrft_denoise_fit(fgfrft_denoise* problem, int epochs, double lr, double init_alpha,
                       double* traj_loss, double* traj_alpha, double* alpha_best, double* h_best,
                       double* loss_best, int* best_epoch, double* reconstruction);
/* Exact backend (ExactDenoiseEngine, learn.hpp:205-289) on a device spectrum, any unitary F:
 * F^a = V diag(e^{j a theta}) V^H, six FP64 tensor-core ZGEMMs per evaluation; loss on the
 * complex residual, or on its real part when loss_on_real. eval / fit / reconstruct / destroy as
 * for the fast backend. */
int fgfrft_denoise_create_exact(fgfrft_spectrum* spectrum, const double* y, const double* x_ref,
                                int64_t channels, int loss_on_real, fgfrft_denoise** out);
/* Re(Q^{-alpha} h o Q^alpha y) at (alpha, h): n x channels real (learn.hpp:232-234, 405-408). */
int fgfrft_denoise_reconstruct(fgfrft_denoise* problem, double alpha, const double* h, double* out);

/* ---- on-disk power cache ----------------------------------------------
 *
 * save: header (magic "FGFRFTC\1", dtype, storage, n, L, fingerprint), F as n x n complex128
 * column-major (the bytes content_fingerprint hashes), the resident slabs as they lie in HBM, and
 * a 64-bit device checksum of the slabs. load: rebuilds the handle without the O(L n^3) build --
 * budget check as in the constructor (FGFRFT_CAPACITY), F re-fingerprinted against the header
 * and the slab checksum re-computed on the device (mismatch -> FGFRFT_NUMERICAL), bad magic /
 * truncation -> FGFRFT_PARSE, open / write failures -> FGFRFT_IO. File IO overlaps the copies
 * through two pinned staging buffers.
 */
int fgfrft_cache_save(fgfrft_cache* cache, const char* path);
int fgfrft_cache_load(const char* path, uint64_t memory_budget, int device, fgfrft_cache** out);

/* ---- spectral form and the exact GFRFT (spectral.hpp:19-195) ------------------------------
 *
 * fgfrft_spectrum holds F = V diag(e^{j theta}) V^H on a device: V n x n complex128, theta
 * ascending in (-pi, pi]. create: a recorded spectrum (KnownSpectrum, gft.hpp:21-25), stored as
 * given. decompose: eigendecompose_unitary (spectral.hpp:121-155) of a host F -- Hermitian part
 * (F + F^H)/2 by cuSOLVER (real F: the real symmetric solver), clusters of cos(theta) within 1e-5
 * rediagonalised against -i (F - F^H)/2, phases from Rayleigh quotients, sorted ascending, and
 * the reconstruction residual checked (> 1e-6 -> FGFRFT_NUMERICAL). theta is returned by
 * spectrum_info (n doubles), V by spectrum_vectors (n x n complex128).
 * exact[_dev]: out[a] = V diag(e^{j a theta}) V^H (FGFRFT_Q, exact_gfrft, spectral.hpp:158-166) or
 * V diag(j theta e^{j a theta}) V^H (FGFRFT_DQ, exact_gfrft_grad, :169-174) for every order; one
 * column scaling and one FP64 tensor-core GEMM per order. out: n_alpha blocks of n x n.
 */
int fgfrft_spectrum_create(const double* v, const double* theta, int64_t n, int device,
                           fgfrft_spectrum** out);
int fgfrft_spectrum_decompose(const double* f, int64_t n, int device, fgfrft_spectrum** out);
int fgfrft_spectrum_destroy(fgfrft_spectrum* spectrum);
int fgfrft_spectrum_info(const fgfrft_spectrum* spectrum, int64_t* n, double* theta);
int fgfrft_spectrum_vectors(fgfrft_spectrum* spectrum, double* v);
int fgfrft_spectrum_set_stream(fgfrft_spectrum* spectrum, void* stream);
int fgfrft_exact(fgfrft_spectrum* spectrum, const double* alphas, int n_alpha, int which, double* out);
int fgfrft_exact_dev(fgfrft_spectrum* spectrum, const double* alphas, int n_alpha, int which,
                     void* out_dev);

/* ---- cascaded transform-order learning (learn.hpp:29-166) ----------------------------------
 *
 * CascadeProblem on the device: Yhat = Q_K ... Q_1 (X = I), target F^{target_order} (exact, from
 * the spectrum), loss = |Yhat - target|_F^2 / N^2, per-layer gradients accumulated in reverse
 * through the product (learn.hpp:72-97). Backend fast: Q_l, dQ_l/dalpha synthesised from `cache`
 * (complex128); exact: cache == NULL, Q_l and dQ_l from the spectrum. All products are FP64
 * tensor-core complex GEMMs; the gradient of layer l is 2/N^2 Re<b prefix_{l-1}^H, dQ_l>.
 * learn: learn_orders (learn.hpp:124-166), Adam (lr, 0.9, 0.999, 1e-8) from init_order for
 * `epochs` steps plus a final evaluation; traj_loss has epochs + 1 entries, traj_alphas
 * (epochs + 1) x depth. Non-finite loss or gradient -> FGFRFT_OPTIMIZER.
 */
typedef struct fgfrft_cascade fgfrft_cascade;
int fgfrft_cascade_create(fgfrft_cache* cache, fgfrft_spectrum* spectrum, double target_order, int depth,
                          fgfrft_cascade** out);
int fgfrft_cascade_destroy(fgfrft_cascade* problem);
int fgfrft_cascade_eval(fgfrft_cascade* problem, const double* alphas, double* loss, double* grad);
int fgfrft_cascade_learn(fgfrft_cascade* problem, double init_order, int epochs, double lr,
                         double* traj_loss, double* traj_alphas, double* final_loss,
                         double* final_alphas);

/* ---- batches of small graphs (BASELINE config 5: fractional specformer) ----------------
 *
 * `graphs` independent GFT matrices (n <= 64, complex128 host input, graph-major), powers
 * 1..l stored per graph in complex64 (built in complex128 on DMMA, then demoted). One CTA per
 * graph. All step-time buffers are device arrays: alphas_dev [graphs][heads] (learnable orders
 * live on the GPU; their sinc coefficients are evaluated on the device), x_dev
 * [graphs][ch][n] complex64 (= per graph an n x ch column-major block), y_dev / g_dev
 * [graphs][heads][ch][n] complex64, dlda_dev [graphs][heads] double.
 *   forward:  Y_gh = Q(alpha_gh; F_g) X_g
 *   dlda:     dL/dalpha_gh = sum_k c'_k(alpha_gh) Re<G_gh, F_g^k X_g>  (G = dL/dconj(Y) convention)
 * heads 1..4, ch 1..64.
 */
int fgfrft_batch_create(const double* fs, int64_t graphs, int64_t n, int l, int device,
                        fgfrft_cache** out);
int fgfrft_batch_destroy(fgfrft_cache* batch);
int fgfrft_batch_set_stream(fgfrft_cache* batch, void* stream);
int fgfrft_batch_forward_dev(fgfrft_cache* batch, const double* alphas_dev, int heads,
                             const void* x_dev, int64_t ch, void* y_dev);
int fgfrft_batch_dlda_dev(fgfrft_cache* batch, const double* alphas_dev, int heads,
                          const void* g_dev, const void* x_dev, int64_t ch, void* dlda_dev);

#ifdef __cplusplus
}
#endif

#endif /* FGFRFT_B200_H */
