// capi_internal.cuh -- shared internals of the C ABI translation units (capi*.cu): kernel
// launcher declarations, error / profiling plumbing, the handle structs and the internal helpers
// one unit calls in another. Not part of the public boundary (include/fgfrft_b200.h is).
#pragma once
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <complex>
#include <dlfcn.h>
#include <numeric>
#include <limits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include <cusolverDn.h>

#include "common.cuh"
#include "fgfrft_b200.h"
#include "oz.cuh"

namespace fgb {
double host_sinc(double);
double host_sinc_deriv(double);
void host_sinc_coeffs(double alpha, int l, double* c, double* dc);
void host_sinc_coeffs_fast(double alpha, int l, double* c, double* dc);  // planning tables only
uint64_t host_fnv1a64(const void* data, size_t nbytes);
template <typename R>
cudaError_t launch_synth(const void* slabs, int n, int l_used, const double* coef_dev, int n_alpha, void* out,
                         cudaStream_t stream);
cudaError_t launch_synth_sweep(const void* slabs, int n, int l_used, const double* coef_dev, int n_alpha, void* out,
                               cudaStream_t stream);
int synth_sweep_max_orders();
cudaError_t launch_rect_to_tiled(const void* src, int64_t ld, int m, int ncols, void* dst, cudaStream_t stream,
                                 bool real);
cudaError_t launch_synth_rows(const void* rowp, const void* colp, int n, int r0, int rows, int l_used,
                              const double* coef_dev, int n_alpha, void* out, cudaStream_t stream, bool real,
                              bool out_complex);
cudaError_t launch_dots_rows(const void* rowp, const void* colp, int n, int r0, int rows, int l, const void* m,
                             int64_t m_stride, int n_alpha, double* partial, double* s_out, cudaStream_t stream,
                             bool real);
size_t dots_rows_partial_elems(int n, int rows, int l, int n_alpha);
cudaError_t launch_batch_coef(const double* alphas_dev, int n_orders, int l, double* coef_dev, cudaStream_t stream,
                              int heads = 0);
size_t batch_coef_bytes(int graphs, int heads, int l);  // the doubles + the tcgen05 kernels' FP32 table
cudaError_t launch_batch_to_tiled(const void* src, int graphs, int n, int l, int k, void* dst, bool real,
                                  cudaStream_t stream);
cudaError_t launch_batch_forward(const void* slabs, int graphs, int n, int l, const double* coef, int heads,
                                 const void* x, int ch, void* y, bool real, cudaStream_t stream);
cudaError_t launch_batch_dlda(const void* slabs, int graphs, int n, int l, const double* coef, int heads,
                              const void* gcot, const void* x, int ch, double* dlda, bool real, cudaStream_t stream);
int batch_max_heads();
int batch_max_channels();
int batch_max_n();
cudaError_t launch_rgemm(int am, int bm, int cm, int M, int N, int K, const void* A, int64_t lda, int64_t sA,
                         const void* B, int64_t ldb, int64_t sB, void* C, int64_t ldc, int64_t sC, int batch,
                         cudaStream_t stream);
cudaError_t launch_rto_tiled(const void* src, void* dst, int n, cudaStream_t stream);
cudaError_t launch_rfrom_tiled(const void* src, void* dst, int n, cudaStream_t stream);
cudaError_t launch_rfrom_tiled_real(const void* src, void* dst, int n, cudaStream_t stream);
size_t rapply_fused_part_elems(int n, int n_alpha);
int rapply_fused_max_cols();
cudaError_t launch_rapply_fused(const void* slabs, int n, int l_used, const double* coef_dev, int coef_ld, int n_alpha,
                                const double* x, int b, double* part, double* y, cudaStream_t stream);
cudaError_t launch_real_part(const void* src, void* dst, int64_t count, cudaStream_t stream);
cudaError_t launch_rsynth(const void* slabs, int n, int l_used, const double* coef_dev, int n_alpha, void* out,
                          bool out_complex, cudaStream_t stream);
cudaError_t launch_rsynth_sweep(const void* slabs, int n, int l_used, const double* coef_dev, int n_alpha, void* out,
                                bool out_complex, cudaStream_t stream);
int rsweep_max_orders();
cudaError_t launch_rdots(const void* slabs, int n, int l, const void* m, int64_t m_stride, int n_alpha, double* partial,
                         double* s_out, cudaStream_t stream);
cudaError_t launch_rdots_mma(const void* slabs, int n, int l, const void* m, int64_t m_stride, int n_alpha,
                             double* partial, double* s_out, cudaStream_t stream, int* launches);
size_t rdots_mma_partial_elems(int n);
cudaError_t launch_zgemm(int M, int N, int K, const void* A, int64_t lda, int64_t sA, bool conj_a, const void* B,
                         int64_t ldb, int64_t sB, bool conj_b, void* C, int64_t ldc, int64_t sC, int batch,
                         bool accumulate, cudaStream_t stream);
cudaError_t launch_power_dots(const void* slabs, int n, int l, const void* m, int64_t m_stride, int n_alpha,
                              double* partial, double* s_out, cudaStream_t stream, int elem_bytes);
cudaError_t launch_cgemm(int M, int N, int K, const void* A, int64_t lda, int64_t sA, bool conj_a, const void* B,
                         int64_t ldb, int64_t sB, bool conj_b, void* C, int64_t ldc, int64_t sC, int batch,
                         bool accumulate, cudaStream_t stream);
cudaError_t launch_promote(const void* src, void* dst, int64_t count, cudaStream_t stream);
// spectral.cu (exact GFRFT, eigendecomposition pieces, cascade reductions)
size_t sp_part_elems();
cudaError_t launch_herm_parts(const void* f, int n, bool real, void* a, void* bh, cudaStream_t st);
cudaError_t launch_real_to_cplx(const double* src, int64_t count, void* dst, cudaStream_t st);
cudaError_t launch_blockdiag(const void* in, int n, const int* colinfo, const void* u, void* out, cudaStream_t st);
cudaError_t launch_col_pair_dot(const void* w, const void* t, int n, const int* pairs, int count, void* out,
                                cudaStream_t st);
cudaError_t launch_gather_cols(const void* src, int n, const int* perm, void* dst, cudaStream_t st);
cudaError_t launch_eig_residual(const void* fw, const void* w, const double* theta, const void* f, int n,
                                double* part, double* out2, cudaStream_t st);
cudaError_t launch_spec_scale(const void* v, const double* theta, const double* alphas, int na, int which, int n,
                              void* w, cudaStream_t st);
cudaError_t launch_cdiff_sq(const void* y, bool real_y, const void* t, int64_t count, void* b, double* part,
                            cudaStream_t st);
cudaError_t launch_cre_dot(const void* m, const void* d, bool real_d, int64_t count, double* part, cudaStream_t st);
cudaError_t launch_sum_parts(const double* part, int groups, double s0, double s1, double* out, cudaStream_t st);
cudaError_t launch_rdot(const double* a, const double* b, int64_t count, double* part, cudaStream_t st);
// store.cu
cudaError_t launch_checksum(const void* data, size_t bytes, unsigned long long* out, cudaStream_t st);
// shard.cu (fused row gather, DMMA path)
cudaError_t launch_rows_push(const void* src, int64_t n, int r0, int rows, int64_t cols, void* const* dst_dev,
                             int ndst, cudaStream_t stream);
size_t dots_partial_elems(int n, int l, int n_alpha);
size_t dots_mma_partial_elems(int n);
int dots_mma_max_orders();
cudaError_t launch_power_dots_mma(const void* slabs, int n, int l, const void* m, int64_t m_stride, int n_alpha,
                                  double* partial, double* s_out, cudaStream_t stream, int* launches);
cudaError_t launch_mse_residual(const void* y, const void* xc, int64_t count, int n_alpha, double g_scale,
                                double loss_scale, void* g, double* partial, double* loss_out, cudaStream_t stream,
                                int elem_bytes);
size_t mse_partial_elems(int n_alpha);
cudaError_t launch_demote(const void* src, void* dst, int64_t count, cudaStream_t stream);
cudaError_t launch_to_tiled(const void* src, void* dst, int n, int elem_bytes_dst, cudaStream_t stream);
cudaError_t launch_from_tiled(const void* src, void* dst, int n, int elem_bytes_src, cudaStream_t stream);
cudaError_t launch_coef_dot(const double* dc, const double* s, int n_alpha, int width, double* out,
                            cudaStream_t stream);
int combine_max_terms();
cudaError_t launch_dn_coef(const double* params, int l, double* tab, cudaStream_t st);
cudaError_t launch_dn_scale(const double* u, const double* h, double* v, int n, int64_t count, cudaStream_t st);
cudaError_t launch_dn_residual(const double* w, const double* x, double* r, int64_t count, double* part,
                               cudaStream_t st);
cudaError_t launch_dn_grad(const double* u, const double* du, const double* h, const double* r, const double* dqhv,
                           const double* qr, int n, int ch, double* grad, double* part, double* loss, int* flag,
                           int epoch, cudaStream_t st);
cudaError_t launch_dn_track(const double* loss, const double* params, int np, int epoch, double* traj, double* best,
                            int* best_epoch, cudaStream_t st);
cudaError_t launch_dnx_phase(const double* params, const double* theta, int n, void* phase, void* jtp, void* jtc,
                             cudaStream_t st);
cudaError_t launch_dnx_rowscale(const void* src, const void* d, const double* h, bool conj_d, int n, int64_t count,
                                void* dst, cudaStream_t st);
cudaError_t launch_dnx_cot(const void* w, const double* x, int64_t count, bool real_loss, void* cot, double* part,
                           cudaStream_t st);
cudaError_t launch_dnx_grad(const void* far, const void* u, const void* vhr, const void* b, const void* jtc,
                            const void* q, const double* h, int n, int ch, double* grad_h, double* part,
                            cudaStream_t st);
cudaError_t launch_dn_finish(const double* part, double* loss, double* grad, int n, int* flag, int epoch,
                             cudaStream_t st);
cudaError_t launch_dn_adam(double* params, double* m, double* v, const double* grad, int np, int64_t step, double lr,
                           cudaStream_t st);
size_t dn_part_elems();
cudaError_t launch_ortho_residual(const double* g, int n, double* out, cudaStream_t stream);
cudaError_t launch_colstats(const double* x, const double* xc, int n, int b, double* colsq, double* colxc, int* ecol,
                            double* rg, int l, cudaStream_t st);
cudaError_t launch_gram_s_dlda(const double* coef, const double* dcoef, const double* rg, int n_alpha, int l,
                               double norm, double* s, double* dlda, cudaStream_t st);
cudaError_t launch_gram_terms(const double* part, int ctas, int tp2, int l, double* rg, cudaStream_t st);
cudaError_t launch_loss3(const double* part, int ctas, int n_alpha, double norm, double* loss, cudaStream_t st);
cudaError_t launch_gram_s(const double* coef, const double* rg, int n_alpha, int l, double norm, double* s,
                          cudaStream_t st);
size_t combine_partial_elems(int tp);
size_t node_partial_elems();
int node_max_terms();
cudaError_t launch_add_diag(double* w, int n, int64_t stride, const double* d, int r, cudaStream_t stream);
cudaError_t launch_node_combine(const double* zin, const double* xc, int64_t count, int r, int rp, const double* pc,
                                int n_alpha, double* y, double* partial, double norm, double* loss, double* dlda,
                                cudaStream_t stream);
cudaError_t launch_combine(int mode, const double* z, const double* x, const double* xc, int64_t count, int l,
                           const double* coef, int n_alpha, double norm, double* y, double* partial, double* s,
                           double* loss, cudaStream_t stream);
// packed.cu (the packed power cache and the one- / two-order step route)
size_t packed_bytes(int n, int l);
cudaError_t launch_pack_tiles(const void* slabs, int n, int l, void* packed, double* scales, cudaStream_t stream,
                              unsigned long long* pmax = nullptr);
// exps[a rp + i] = the Ozaki row exponent of a bound on |(Q_a - c_0 I)[i, :]| from the power maxima
cudaError_t launch_prow_bound(const unsigned long long* pmax, int n, int l, const double* coef, int coef_ld, int ac,
                              int rp, int* exps, cudaStream_t stream);
// the order window (packed.cu): Q_x = sum_j w[x][j] W'_j over r <= kWindowMaxNodes node operators
cudaError_t launch_window_synth(const double* wops, int r, int n, const WindowWeights& ww, int rows, double* out,
                                int64_t ostride, unsigned long long* rowmax, int64_t mp, cudaStream_t stream,
                                int row0 = 0, int row1 = -1);
cudaError_t launch_psynth(const void* packed, const double* scales, int n, int l, int l_cache, const double* coef_dev,
                          int coef_ld, int n_alpha, double* out, int64_t out_stride, unsigned long long* rowmax,
                          int64_t rm_stride, cudaStream_t stream, int p0 = 0, int p1 = -1, int max_ctas = 0,
                          int pbase = 0, int nodiag = 0, int8_t* digits = nullptr, const int* exps = nullptr,
                          int rp = 0, int kp = 0, int sd = 0);
cudaError_t launch_pack_pairs_from_panels(const double* rp, int64_t ld_r, const double* cp, int64_t ld_c, int n, int I0,
                                          int pbase, int npairs_local, int k, int l, void* packed, double* scales,
                                          cudaStream_t stream);
size_t packed_bytes_pairs(int64_t npairs, int l);
cudaError_t launch_sum_slots(const double* slots, int nslots, int64_t count, double* out, cudaStream_t stream);
size_t packed_scale_elems(int n, int l);
int64_t packed_pairs_before(int I, int nt);
size_t mse_dy_part_elems();
// The fused-MSE product GEMM's partials (OzOut::lpart): order a owns the slot run [a per, (a + 1) per)
// of (loss, dot) pairs, per = Y tiles of one block x 16 epilogue warps; loss = sum * norm, dL/da = 2 dot norm.
cudaError_t launch_fused_mse_finish(const double* part, int64_t per, int n_alpha, double norm, double* loss,
                                    double* dlda, cudaStream_t stream);
cudaError_t launch_mse_dy(const void* y, const void* dy, const void* xc, int64_t count, void* yout, double* part,
                          double norm, double* loss, double* dlda, cudaStream_t stream);
cudaError_t launch_mse_dy_part(const void* y, const void* dy, const void* xc, int64_t count, void* yout, double* part,
                               int slot, cudaStream_t stream);
cudaError_t launch_mse_dy_finish_n(const double* part, int nslots, double norm, double* loss, double* dlda,
                                   cudaStream_t stream);
}  // namespace fgb

using namespace fgb;

namespace fgbi {

extern thread_local std::string g_err;
// Set by the host-buffer entry points around their call into a *_dev entry point: the device
// buffers they pass are already in the internal (complex128) layout, no complex64 bridge.
extern thread_local bool tl_internal_signals;
struct InternalSignals {
    bool prev;
    InternalSignals() : prev(tl_internal_signals) { tl_internal_signals = true; }
    ~InternalSignals() { tl_internal_signals = prev; }
};
extern std::atomic<uint64_t> g_launches;

// Optional per-kernel-class timing with CUDA events recorded on the launching stream
// (fgfrft_profile_*): bench.py uses it to time the dominant kernel inside its timed region.
enum KernelClass {
    KC_SYNTH = 0, KC_GEMM = 1, KC_DOTS = 2, KC_ELEMWISE = 3, KC_I8GEMM = 4, KC_SLICE = 5, KC_COMBINE = 6, KC_NODEOP = 7, KC_COUNT = 8
};
struct ProfRec {
    int cls;
    cudaEvent_t a, b;
};
extern std::mutex g_prof_mu;
extern bool g_prof_on;
extern std::vector<ProfRec> g_prof;
extern std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event();

struct ProfScope {
    int cls;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    ProfScope(int c, cudaStream_t s) : cls(c), st(s) {
        if (!g_prof_on) return;
        std::lock_guard<std::mutex> lk(g_prof_mu);
        a = prof_event();
        cudaEventRecord(a, st);
    }
    ~ProfScope() {
        if (!a) return;
        std::lock_guard<std::mutex> lk(g_prof_mu);
        cudaEvent_t b = prof_event();
        cudaEventRecord(b, st);
        g_prof.push_back({cls, a, b});
    }
};

int fail(int code, const std::string& msg);

#define FGB_CUDA(expr)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (expr);                                                                \
        if (e_ != cudaSuccess) {                                                                \
            cudaGetLastError();                                                                 \
            return fail(FGFRFT_CUDA, std::string(#expr) + " failed: " + cudaGetErrorString(e_)); \
        }                                                                                       \
    } while (0)

#define FGB_LAUNCH(expr, nlaunch)  \
    do {                           \
        FGB_CUDA(expr);            \
        g_launches += (nlaunch);   \
    } while (0)

#define FGB_GUARD_BEGIN try {
#define FGB_GUARD_END                                                        \
    }                                                                        \
    catch (const std::bad_alloc&) {                                          \
        return fail(FGFRFT_CAPACITY, "host allocation failed");              \
    }                                                                        \
    catch (const std::exception& ex) {                                       \
        return fail(FGFRFT_NUMERICAL, ex.what());                            \
    }                                                                        \
    catch (...) {                                                            \
        return fail(FGFRFT_NUMERICAL, "unknown exception");                  \
    }

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

}  // namespace fgbi

using namespace fgbi;

// One row shell of the pipelined packed route (capi.cu packed_products).
struct PkShell {
    int r0, r1;  // rows [r0, r1)
    int p0, p1;  // I-major tile pairs [p0, p1)
};

struct fgfrft_cache {
    int64_t n = 0;
    int l = 0;
    int dtype = FGFRFT_C128;
    bool real = false;  // F has an exactly zero imaginary part: real cache, real Q, real x complex GEMMs
    // complex64 API over a real F: the powers are stored as real doubles (the same 8 bytes per
    // element as complex64) and every kernel runs the real complex128 path; the *_dev entry points
    // promote the caller's complex64 signals on entry and demote the results (dtype stays C128
    // internally, fgfrft_cache_info reports C64).
    bool api_c64 = false;
    DevBuf bx, bxc, by;
    // Node route of order sweeps (real F): the stacked cache as element-row INT8 digit slices
    // (built once), the per-call node coefficient table / interpolation weights, the node
    // operators W_j and their products Z'_j = W_j X.
    int last_route = -1, last_nodes = 0;  // route of the last sweep (fgfrft_cache_route_info)
    int es_slices = 0;
    bool es_pairs = false;  // es holds element-PAIR rows (pair-major, L terms per element) instead of element rows
    DevBuf es, ee, erm, nd_tab, nd_p, nd_d0, nd_bsl, nd_bex, nd_w, nd_z;
    // pinned staging of the per-call node tables: a ring of 3, so the host plans and stages the next
    // calls while the device still runs this one (a single buffer made every call wait for the
    // previous call's GEMMs, exposing the host planning on the device timeline)
    static constexpr int kNdRing = 3;
    double* nd_h = nullptr;  // the current slot's buffer
    double* nd_hr[kNdRing] = {};
    size_t nd_hr_cap[kNdRing] = {};
    cudaEvent_t nd_evr[kNdRing] = {};
    int nd_slot = 0;
    std::vector<double> nd_ctab;  // the sweep's [c | c'] tables for the node plan's check (host)
    struct NodePlan {  // memoised plan of the last sweep (a pure function of the orders)
        std::vector<double> alphas, tab, d0, pw;
        int hint_r = 0;  // node count of the last accepted plan, its width: the next search's start
        double hint_w = 0.0;
        bool hint_need_d = false;
        bool need_d = false, ok = false;
        bool staged = false;  // tab / d0 / pw of this plan already resident in nd_tab / nd_d0 / nd_p
        int r = 0, rp = 0;
    } nd_plan;
    size_t sig = 16;    // bytes per signal element (X, Y, G): 16 complex128, 8 complex64
    int device = 0;
    uint64_t fingerprint = 0;
    void* slabs = nullptr;
    size_t elem = 16;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    std::mutex mu;
    // workspaces
    DevBuf coef, q, m, partial, s, x, y, g, xc, lpart, loss, dlda, tmp;
    // Power-product route (real F): the stacked cache [P_1..P_L; P_1^T..P_L^T] as INT8 Ozaki
    // digit slices (built lazily, once), the per-call slices of X and the products Z = P X.
    int engine = FGFRFT_ENGINE_AUTO;
    // F^T F = I to rounding (unitarity residual of gft.hpp:39-44 <= 1e-12, checked on device at
    // build): the power-product MSE step may then take s_k from the Gram sequence <X, F^d X>.
    bool orthogonal = false;
    double ortho_residual = -1.0;
    int ps_slices = 0;
    DevBuf ps, pe, prm, xsl, xex, z;
    DevBuf qsl, qex;  // per-call INT8 slices of Q(a) (or G) for the synthesis route
    // Orthogonal-F sweep with the combination on the INT8 tensor cores: the stacked cache sliced
    // in (signal row, term) interleaved order, P_L in column-major form, and per-call buffers.
    int ps3_slices = 0;
    DevBuf ps3, pe3, plr, zd, zaux, cdig, cex;
    // Pair shard (fgfrft_pshard_*, capi_pshard.cu): tile pairs [pbase, pend) = tile-row band
    // [I0, I1) of `world`; the packed slabs (pk, pks) hold only those pairs; pp = this rank's
    // partial [Y; dY] (zero outside its rows), ppc = the reduce-scatter's column chunk.
    bool pshard = false;
    int world = 1, rank = 0, I0 = 0, I1 = 0;
    int64_t pbase = 0, pend = 0;
    struct fgfrft_comm* comm = nullptr;
    DevBuf pp, ppc;
    int64_t pp_b = -1;
    int pp_rows = -1;
    // fused reduce-scatter: rb = this rank's receive slots [source rank][rows blocks][n x cb complex];
    // rb_dest = every owner's slot for this rank (peers mapped through CUDA IPC), rb_open = mappings
    DevBuf rb, bar;
    std::vector<double*> rb_dest;
    std::vector<void*> rb_open, rb_peer;
    void* rb_for = nullptr;
    // Row-slab shard (fgfrft_shard_*): rows [r0, r1); slabs = row panels, colp = column panels.
    bool shard = false;
    int64_t graphs = 0;  // > 0: batch of small graphs (fgfrft_batch_*), n <= 64, complex64
    int64_t r0 = 0, r1 = 0;
    void* colp = nullptr;
    size_t panel_elems = 0;
    // Host-buffer MSE step: Xc is uploaded on a side stream while the power products run; the
    // step waits on xc_evt right before its first use of Xc.
    cudaStream_t aux_stream = nullptr;
    cudaEvent_t xc_evt = nullptr;
    bool xc_pending = false;
    // Memory budget of the handle (transform.hpp:46-53 counts L n^2 16 bytes): auxiliary device
    // representations (packed slabs, INT8 digit slices) are built only while the reference count
    // plus their bytes stays within it; otherwise the routes that need them are not taken.
    uint64_t budget = 0;
    uint64_t aux_bytes = 0;
    // Packed power cache (packed.cu): 40-bit fixed-point tiles + per-tile scales, for the one- /
    // two-order step and apply route (real F). 0 not built, 1 ready, -1 unavailable.
    int pk_state = 0;
    DevBuf pk, pks, ydy;
    DevBuf pkm;  // [L][2][32 nt] row / column maxima of the powers (digit-emitting synthesis; empty: off)
    // Digit cache of the INT8 tensor-core synthesis (ozgemm.cu dsynth_kernel): pair-major element
    // rows x powers, 5 base-254 digits + one exponent per element row; the coefficient digits.
    // Replaces the packed slabs on the step route when it fits. 0 not built, 1 ready, -1 unavailable.
    int ds_state = 0;
    bool pk_tc = false;  // the last packed_products synthesised on the tensor cores
    bool pk_emit = false;  // the last packed_products' synthesis emitted Q's digits (no slicing pass)
    // the order window (fgfrft_cache_set_order_window): r exact FP64 node operators W'_j (c_0 I left
    // out) at the Chebyshev nodes of [win_lo, win_hi]; the step route synthesises Q, dQ/da of orders
    // inside it from these instead of the packed powers
    DevBuf win;
    int win_r = 0;
    double win_lo = 0.0, win_hi = 0.0;
    std::vector<double> win_xn, win_bw;
    bool pk_win = false;  // the last packed_products synthesised from the window
    DevBuf ds, dse, dsb;
    // shell pipeline of the packed route: side streams (S synthesis + slicing, G GEMMs, high
    // priority), fork / join events, one event per shell, the memoised shell plan
    cudaStream_t pk_s = nullptr, pk_g = nullptr;
    cudaEvent_t pk_e0 = nullptr, pk_eg = nullptr, pk_ex = nullptr;
    // node route: the last node-operator GEMM has read the coefficient digits / diagonal (the next
    // call's tables may overwrite them on the side stream), and this call's digits are ready
    cudaEvent_t nd_ev_op = nullptr, nd_ev_b = nullptr;
    std::vector<cudaEvent_t> pk_es;
    std::vector<cudaEvent_t> xh_ev;  // host-X column chunks landed (chunked host MSE step)
    std::vector<cudaEvent_t> xch_ev; // host-Xc column chunks landed (the loss pass runs per chunk)
    const double* xh_pre = nullptr;  // host X whose chunk copies the caller already enqueued (enqueue_host_x)
    std::vector<PkShell> pk_plan;
    uint64_t pk_plan_key = 0;
    // pinned staging for the coefficient tables: a ring of 3 (the host evaluates the next calls'
    // tables while this call's upload is queued behind the device's work); coef_h = current slot
    static constexpr int kCoefRing = 3;
    double* coef_h = nullptr;
    double* coef_hr[kCoefRing] = {};
    size_t coef_hr_cap[kCoefRing] = {};
    cudaEvent_t coef_evr[kCoefRing] = {};
    int coef_slot = 0;
    std::vector<double> coef_alphas;  // orders of the tables now in `coef` / coef_h (memo)
    int coef_l = -1;

    // Matrices at the API are n x n column-major; device slabs are tiled (common.cuh) and padded
    // to npad = 32 * ceil(n / 32) per side.
    size_t mat_elems() const { return (size_t)n * (size_t)n; }
    size_t npad() const { return (size_t)ceil_div(n, kTile) * kTile; }
    size_t slab_elems() const { return npad() * npad(); }
    size_t slab_bytes() const { return slab_elems() * elem; }
    void* slab(int k) const { return static_cast<char*>(slabs) + (size_t)(k - 1) * slab_bytes(); }
};

struct fgfrft_denoise {
    fgfrft_cache* cache = nullptr;
    int64_t n = 0, ch = 0, cpad = 0;
    int l = 0;
    DevBuf y, x, qd, uu, ww, qr, v, r, params, grad, adam, tab, part, scal, best, traj, flag;  // qd = [Q | dQ]
    // exact backend (learn.hpp:205-289): the spectrum and its n x ch complex blocks
    fgfrft_spectrum* spec = nullptr;
    bool exact = false, loss_on_real = false;
    bool cplx = false;  // fast backend over a complex F: complex blocks in the x* buffers
    DevBuf xytil, xu, xb, xw, xcot, xvhr, xfar, xq, xt, xph;
};

struct fgfrft_spectrum {
    int64_t n = 0;
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    std::mutex mu;
    DevBuf v, theta, alph, w;
    std::vector<double> theta_h;
};

struct fgfrft_cascade {
    fgfrft_cache* cache = nullptr;  // fast backend; nullptr: exact backend through the spectrum
    fgfrft_spectrum* spec = nullptr;
    int k = 0;
    int64_t n = 0;
    DevBuf target, ops, dops, prefix, b, nb, m, part, out;
    cudaStream_t stream() const { return cache ? cache->stream : spec->stream; }
};

namespace fgbi {

// helpers defined in one capi*.cu unit and used in another
int ensure_power_slices(fgfrft_cache* c);
int64_t pad_k(int64_t n);
int64_t pad_rows(int64_t n);
int zgemm_auto(int opa, int opb, int64_t m, int64_t n, int64_t k, const void* a, int64_t lda, int64_t sa,
               const void* b, int64_t ldb, int64_t sb, void* c, int64_t ldc, int64_t sc, int batch, cudaStream_t st);
int check_handle(const fgfrft_cache* c);
void destroy_cache(fgfrft_cache* c);
int check_shard(const fgfrft_cache* c);
int check_alphas(const double* alphas, int n_alpha);
int upload_coefs(fgfrft_cache* c, const double* alphas, int n_alpha, int l, double** dev);
bool use_int8_gemm(const fgfrft_cache* c, int64_t b);
int int8_qx_gen(fgfrft_cache* c, int na, bool inverse, const void* q, int64_t m, int64_t ldq, int64_t sq,
                const void* x_dev, int64_t b, void* y, int64_t ldy, int64_t sy, double* const* peers = nullptr,
                int npeers = 0, bool rowmax_ready = false, cudaEvent_t x_sliced = nullptr, int64_t x_bp = 0);
int int8_gx_gen(fgfrft_cache* c, int na, const void* g, int64_t m, const void* x_dev, int64_t b, void* out,
                int64_t sm);
int check_batch(const fgfrft_cache* c);
int synth_into(fgfrft_cache* c, const double* coef_dev, int n_alpha, int l_used, void* out, bool internal = false);
int int8_qx(fgfrft_cache* c, int na, bool inverse, const void* q, const void* x_dev, int64_t b, void* y,
            bool rowmax_ready = false, cudaEvent_t x_sliced = nullptr, int64_t x_bp = 0);
int create_common(const double* f, int64_t n, int l, uint64_t budget, int dtype, int device, fgfrft_cache** out,
                  fgfrft_cache** made);
int check_orthogonal(fgfrft_cache* c, const double* fr, double* scratch);
int check_spectrum(const fgfrft_spectrum* s);
bool aux_fits(const fgfrft_cache* c, uint64_t bytes);
int wait_xc(fgfrft_cache* c);
bool packed_enabled(const fgfrft_cache* c);
uint64_t power_slice_bytes(const fgfrft_cache* c);
uint64_t elem_slice_bytes(const fgfrft_cache* c);
int ensure_elem_slices(fgfrft_cache* c);
bool ensure_packed(fgfrft_cache* c);
bool ensure_dsynth(fgfrft_cache* c);
bool ensure_step_cache(fgfrft_cache* c);
int packed_products(fgfrft_cache* c, const double* coef, int coef_ld, int rows, const void* x_dev, int64_t b,
                    void* y, int l_used, const double* x_host = nullptr, const WindowWeights* ww = nullptr,
                    const double* fuse_xc = nullptr, double* fuse_part = nullptr, bool* fused = nullptr);
// slots the fused-MSE product GEMM writes per order (launch_fused_mse_finish's per), in double2
int64_t fused_mse_slots_per_order(int64_t n, int64_t b);
// true (and the weights rows [l_j(a) ..][l_j'(a) ..] when with_d) when every order lies in the window
bool window_weights(const fgfrft_cache* c, const double* alphas, int n_alpha, bool with_d, int l_used,
                    WindowWeights* ww);
int mse_packed_step(fgfrft_cache* c, const double* coef, int n_alpha, const void* x_dev, const void* xc_dev, int64_t b,
                    void* y_dev, double* loss_dev, double* dlda_dev, const WindowWeights* ww = nullptr,
                    const double* x_host = nullptr,
                    const double* xc_host = nullptr);

}  // namespace fgbi
