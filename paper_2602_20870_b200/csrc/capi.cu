// capi.cu -- the C ABI (include/fgfrft_b200.h): handle lifetime, validation with the
// reference's error semantics, host<->device staging and orchestration of the kernels.
//
// Reference interfaces replaced (proj/include/fgfrft/):
//   PowerCache ctor / power / verify / fingerprint  transform.hpp:43-74   -> fgfrft_cache_*
//   fgfrft_matrix / fgfrft_grad                     transform.hpp:111-136 -> fgfrft_synthesize*
//   apply_forward / apply_inverse                   transform.hpp:138-148 -> fgfrft_apply*, _matrix
//   sinc_coeffs                                     sinc.hpp:50-63        -> fgfrft_sinc_coeffs
//   dL/dalpha contraction                           learn.hpp:88-94       -> fgfrft_dlda*, mse_step*
// plus the INT8 engine entry points (fgfrft_dgemm_int8_dev, fgfrft_zgemm_int8_dev). The other C-ABI
// units: capi_shard.cu (row shards, fused gather, graph batches), capi_learn.cu (denoising
// learner), capi_spectral.cu (spectrum, exact GFRFT, cascade), capi_store.cu (on-disk cache);
// shared internals in capi_internal.cuh.
#include "capi_internal.cuh"

namespace fgbi {

// Host-side time of the per-call planning stages (FGFRFT_HOST_PROF=1: printed at exit) -- the order
// sweeps' host work must stay under their device time or the device idles between calls.
struct HostProf {
    const bool on = [] {
        const char* e = std::getenv("FGFRFT_HOST_PROF");
        return e && std::atoi(e) == 1;
    }();
    double t[8] = {};
    long n[8] = {};
    ~HostProf() {
        if (!on) return;
        static const char* names[8] = {"upload_coefs", "node_plan", "node_stage", "node_products", "combine",
                                       "mse_step_dev", "", ""};
        for (int k = 0; k < 8; ++k)
            if (n[k]) std::fprintf(stderr, "[fgfrft host] %-14s %8.1f us/call (%ld calls)\n", names[k], t[k] / n[k] * 1e6, n[k]);
    }
};
static HostProf g_hprof;
struct HostTimer {
    int k;
    std::chrono::steady_clock::time_point t0;
    explicit HostTimer(int k_) : k(k_) {
        if (g_hprof.on) t0 = std::chrono::steady_clock::now();
    }
    ~HostTimer() {
        if (!g_hprof.on) return;
        g_hprof.t[k] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        ++g_hprof.n[k];
    }
};

thread_local std::string g_err;
thread_local bool tl_internal_signals = false;
std::atomic<uint64_t> g_launches{0};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event() {
    if (!g_prof_pool.empty()) {
        cudaEvent_t e = g_prof_pool.back();
        g_prof_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

}  // namespace fgbi

namespace fgbi {

int check_handle(const fgfrft_cache* c) {
    if (!c) return fail(FGFRFT_PARAMETER, "null fgfrft_cache handle");
    if (c->shard) return fail(FGFRFT_PARAMETER, "row-shard handle: use the fgfrft_shard_* entry points");
    if (c->pshard) return fail(FGFRFT_PARAMETER, "pair-shard handle: use the fgfrft_pshard_* entry points");
    if (c->graphs > 0) return fail(FGFRFT_PARAMETER, "graph-batch handle: use the fgfrft_batch_* entry points");
    return FGFRFT_OK;
}

int check_batch(const fgfrft_cache* c) {
    if (!c) return fail(FGFRFT_PARAMETER, "null fgfrft_batch handle");
    if (c->graphs <= 0) return fail(FGFRFT_PARAMETER, "not a graph-batch handle");
    return FGFRFT_OK;
}

int check_shard(const fgfrft_cache* c) {
    if (!c) return fail(FGFRFT_PARAMETER, "null fgfrft_shard handle");
    if (!c->shard || c->graphs > 0) return fail(FGFRFT_PARAMETER, "not a row-shard handle");
    return FGFRFT_OK;
}

// Orders per device chunk: keep a chunk's Q / M workspace L2-resident (~64 MiB) when possible.
int alpha_chunk(const fgfrft_cache* c, int n_alpha) {
    if (const char* env = std::getenv("FGFRFT_ALPHA_CHUNK")) {
        const int v = std::atoi(env);
        if (v > 0) return v < n_alpha ? v : n_alpha;
    }
    // All orders of a sweep in one chunk up to ~4 GiB of Q / M workspace: the synthesis and
    // power-dot kernels then stream the cache from HBM once per call.
    const size_t budget = (size_t)4 << 30;
    size_t a = budget / (c->mat_elems() * 16);
    if (a < 1) a = 1;
    if (a > (size_t)n_alpha) a = (size_t)n_alpha;
    return (int)a;
}

// Compute [c | dc] tables for the orders (layout [2][n_alpha][2l+1]) into pinned memory and
// upload them on the handle stream. The previous upload must have completed before the
// pinned staging is rewritten (it is enqueued ahead of the kernels that read it).
int upload_coefs(fgfrft_cache* c, const double* alphas, int n_alpha, int l, double** dev) {
    const size_t width = (size_t)(2 * l + 1);
    const size_t count = 2 * (size_t)n_alpha * width;
    if (c->coef_l == l && c->coef_alphas.size() == (size_t)n_alpha &&
        !std::memcmp(c->coef_alphas.data(), alphas, (size_t)n_alpha * sizeof(double))) {
        *dev = c->coef.as<double>();  // same orders as the tables already on the device: no host work
        return FGFRFT_OK;
    }
    c->coef_l = -1;
    const int q = (c->coef_slot + 1) % fgfrft_cache::kCoefRing;
    if (c->coef_evr[q]) FGB_CUDA(cudaEventSynchronize(c->coef_evr[q]));  // its upload, kCoefRing calls ago
    if (c->coef_hr_cap[q] < count) {
        if (c->coef_hr[q]) cudaFreeHost(c->coef_hr[q]);
        c->coef_hr[q] = nullptr;
        c->coef_hr_cap[q] = 0;
        FGB_CUDA(cudaMallocHost(&c->coef_hr[q], count * sizeof(double)));
        c->coef_hr_cap[q] = count;
    }
    c->coef_slot = q;
    c->coef_h = c->coef_hr[q];
    // 2 (2L+1) libm evaluations per order, on this thread: an OpenMP team here measured 1.4 ms per
    // call inside a process whose other OpenMP pools spin (CPU quota), against 0.05 ms alone -- and
    // the order sweeps, whose host planning would need it, plan from host_sinc_coeffs_fast tables
    for (int a = 0; a < n_alpha; ++a)
        host_sinc_coeffs(alphas[a], l, c->coef_h + a * width, c->coef_h + ((size_t)n_alpha + a) * width);
    FGB_CUDA(c->coef.ensure(count * sizeof(double)));
    FGB_CUDA(cudaMemcpyAsync(c->coef.p, c->coef_h, count * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    if (!c->coef_evr[q]) FGB_CUDA(cudaEventCreateWithFlags(&c->coef_evr[q], cudaEventDisableTiming));
    FGB_CUDA(cudaEventRecord(c->coef_evr[q], c->stream));
    c->coef_alphas.assign(alphas, alphas + n_alpha);
    c->coef_l = l;
    *dev = c->coef.as<double>();
    return FGFRFT_OK;
}

int check_alphas(const double* alphas, int n_alpha) {
    if (n_alpha < 1 || !alphas) return fail(FGFRFT_PARAMETER, "need at least one order");
    for (int a = 0; a < n_alpha; ++a)
        if (!std::isfinite(alphas[a])) return fail(FGFRFT_PARAMETER, "order alpha must be finite");
    return FGFRFT_OK;
}

// Q for n_alpha orders into out (n x n each). Up to 4 orders: exact scalar tile-pair kernel
// (HBM-bound, bit-identical to the reference order of operations). Sweeps of >= 8 complex128
// orders: DMMA kernel, 64 orders per launch, cache streamed once per launch.
int synth_into(fgfrft_cache* c, const double* coef_dev, int n_alpha, int l_used, void* out, bool internal) {
    ProfScope ps(KC_SYNTH, c->stream);
    if (c->real) {  // complex output (imag 0) for the API, real Q for the internal GEMMs
        const bool oc = !internal;
        const size_t oe = oc ? 16 : 8;
        if (n_alpha >= 8 && std::getenv("FGFRFT_EXACT_SWEEP") == nullptr) {
            const int width = 2 * l_used + 1, cap = rsweep_max_orders();
            for (int a0 = 0; a0 < n_alpha; a0 += cap) {
                const int na = std::min(cap, n_alpha - a0);
                FGB_LAUNCH(launch_rsynth_sweep(c->slabs, (int)c->n, l_used, coef_dev + (size_t)a0 * width, na,
                                               static_cast<char*>(out) + (size_t)a0 * c->mat_elems() * oe, oc,
                                               c->stream),
                           1);
            }
        } else {
            FGB_LAUNCH(launch_rsynth(c->slabs, (int)c->n, l_used, coef_dev, n_alpha, out, oc, c->stream), 1);
        }
        return FGFRFT_OK;
    }
    if (c->dtype == FGFRFT_C128 && n_alpha >= 8 && std::getenv("FGFRFT_EXACT_SWEEP") == nullptr) {
        const int width = 2 * l_used + 1;
        const int cap = synth_sweep_max_orders();
        for (int a0 = 0; a0 < n_alpha; a0 += cap) {
            const int na = std::min(cap, n_alpha - a0);
            FGB_LAUNCH(launch_synth_sweep(c->slabs, (int)c->n, l_used, coef_dev + (size_t)a0 * width, na,
                                          static_cast<double2*>(out) + (size_t)a0 * c->mat_elems(), c->stream),
                       1);
        }
        return FGFRFT_OK;
    }
    if (c->dtype == FGFRFT_C128)
        FGB_LAUNCH(launch_synth<double>(c->slabs, (int)c->n, l_used, coef_dev, n_alpha, out, c->stream), 1);
    else
        FGB_LAUNCH(launch_synth<float>(c->slabs, (int)c->n, l_used, coef_dev, n_alpha, out, c->stream), 1);
    return FGFRFT_OK;
}


int create_common(const double* f, int64_t n, int l, uint64_t budget, int dtype, int device, fgfrft_cache** out,
                  fgfrft_cache** made) {
    if (!out) return fail(FGFRFT_PARAMETER, "null output handle pointer");
    *out = nullptr;
    if (l < 1) return fail(FGFRFT_PARAMETER, "PowerCache: truncation order must be >= 1");
    if (n < 1 || !f) return fail(FGFRFT_PARAMETER, "PowerCache: matrix must be non-empty");
    if (n > (1 << 30) / 2) return fail(FGFRFT_CAPACITY, "PowerCache: n exceeds the 32-bit tile index range");
    if (dtype != FGFRFT_C128 && dtype != FGFRFT_C64) return fail(FGFRFT_PARAMETER, "unknown dtype");
    if (dtype == FGFRFT_C64 && (n % 2) != 0)
        return fail(FGFRFT_PARAMETER, "complex64 caches need an even n (16-byte TMA column alignment)");
    const uint64_t elem = dtype == FGFRFT_C128 ? 16 : 8;
    const unsigned __int128 bytes = (unsigned __int128)l * (uint64_t)n * (uint64_t)n * elem;
    if (bytes > budget) {
        std::ostringstream msg;
        msg << "PowerCache: " << l << " powers of a " << n << "x" << n << " matrix need "
            << (unsigned long long)bytes << " bytes, over the " << budget << "-byte budget";
        return fail(FGFRFT_CAPACITY, msg.str());
    }
    int ndev = 0;
    FGB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(FGFRFT_PARAMETER, "device index out of range");
    auto* c = new fgfrft_cache();
    c->n = n;
    c->l = l;
    c->budget = budget;
    c->dtype = dtype;
    c->device = device;
    c->elem = elem;
    c->sig = elem;
    c->fingerprint = host_fnv1a64(f, (size_t)n * (size_t)n * 16);
    if (std::getenv("FGFRFT_NO_REAL") == nullptr) {
        bool real = true;
        for (size_t i = 0; i < (size_t)n * (size_t)n && real; ++i) real = f[2 * i + 1] == 0.0;
        if (real) {
            c->real = true;
            c->elem = 8;
            if (dtype == FGFRFT_C64) {  // same 8 bytes per element, FP64 real kernels (see api_c64)
                c->api_c64 = true;
                c->dtype = FGFRFT_C128;
                c->sig = 16;
            }
        }
    }
    DeviceGuard dg(device);
    cudaError_t e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return fail(FGFRFT_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    c->stream = c->own_stream;
    const size_t alloc = c->slab_bytes() * (size_t)l;
    e = cudaMalloc(&c->slabs, alloc);
    if (e != cudaSuccess) {
        cudaGetLastError();
        cudaStreamDestroy(c->own_stream);
        delete c;
        std::ostringstream msg;
        msg << "PowerCache: device allocation of " << (unsigned long long)alloc
            << " bytes failed (" << cudaGetErrorString(e) << ")";
        return fail(FGFRFT_CAPACITY, msg.str());
    }
    *made = c;
    return FGFRFT_OK;
}

void destroy_cache(fgfrft_cache* c) {
    if (!c) return;
    DeviceGuard dg(c->device);
    if (c->own_stream) cudaStreamSynchronize(c->own_stream);
    if (c->stream != c->own_stream) cudaStreamSynchronize(c->stream);
    if (c->aux_stream) cudaStreamSynchronize(c->aux_stream);
    for (cudaEvent_t e : c->pk_es) cudaEventDestroy(e);
    for (cudaEvent_t e : c->xh_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : c->xch_ev) cudaEventDestroy(e);
    for (void* p : c->rb_open) cudaIpcCloseMemHandle(p);
    for (cudaEvent_t e : {c->pk_e0, c->pk_eg, c->pk_ex, c->nd_ev_op, c->nd_ev_b})
        if (e) cudaEventDestroy(e);
    if (c->pk_s) cudaStreamSynchronize(c->pk_s);
    if (c->pk_g) cudaStreamSynchronize(c->pk_g);
    for (DevBuf* b : {&c->coef, &c->q, &c->m, &c->partial, &c->s, &c->x, &c->y, &c->g, &c->xc, &c->lpart,
                      &c->loss, &c->dlda, &c->tmp, &c->ps, &c->pe, &c->prm, &c->xsl, &c->xex, &c->z, &c->qsl,
                      &c->qex, &c->ps3, &c->pe3, &c->plr, &c->zd, &c->zaux, &c->cdig, &c->cex, &c->bx, &c->bxc,
                      &c->by, &c->es, &c->ee, &c->erm, &c->nd_tab, &c->nd_p, &c->nd_d0, &c->nd_bsl, &c->nd_bex,
                      &c->nd_w, &c->nd_z, &c->pk, &c->pks, &c->ds, &c->dse, &c->dsb, &c->win, &c->ydy, &c->pp, &c->ppc, &c->rb, &c->bar})
        b->release();
    for (int q = 0; q < fgfrft_cache::kCoefRing; ++q) {
        if (c->coef_hr[q]) cudaFreeHost(c->coef_hr[q]);
        if (c->coef_evr[q]) cudaEventDestroy(c->coef_evr[q]);
    }
    for (int q = 0; q < fgfrft_cache::kNdRing; ++q) {
        if (c->nd_hr[q]) cudaFreeHost(c->nd_hr[q]);
        if (c->nd_evr[q]) cudaEventDestroy(c->nd_evr[q]);
    }
    if (c->xc_evt) cudaEventDestroy(c->xc_evt);
    if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
    if (c->pk_s) cudaStreamDestroy(c->pk_s);
    if (c->pk_g) cudaStreamDestroy(c->pk_g);
    if (c->slabs) cudaFree(c->slabs);
    if (c->colp) cudaFree(c->colp);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
}

// Device cache build: P_1 = F, P_k = F P_{k-1} (transform.hpp:57-58) with the DMMA GEMM in
// column-major complex128 scratch, each power then written to its tiled slab (demoted to
// complex64 for C64 caches, so the error does not compound through a complex64 recursion).
// ||F^T F - I||_F / sqrt(n) on the device (2 n^3 DMMA flops, once per cache; real F only).
int check_orthogonal(fgfrft_cache* c, const double* fr, double* scratch) {
    const int n = (int)c->n;
    FGB_LAUNCH(launch_rgemm(1, 0, 0, n, n, n, fr, n, 0, fr, n, 0, scratch, n, 0, 1, c->stream), 1);
    FGB_CUDA(c->lpart.ensure(sizeof(double)));
    FGB_LAUNCH(launch_ortho_residual(scratch, n, c->lpart.as<double>(), c->stream), 1);
    double r2 = 0.0;
    FGB_CUDA(cudaMemcpyAsync(&r2, c->lpart.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    c->ortho_residual = std::sqrt(r2 / (double)n);
    c->orthogonal = c->ortho_residual <= 1e-12;
    return FGFRFT_OK;
}

int build_powers(fgfrft_cache* c, const double* f) {
    const size_t ml = c->mat_elems();
    const int n = (int)c->n;
    if (c->real) {  // P_k = F P_{k-1} as a real DMMA GEMM (2 n^3 flops per power)
        FGB_CUDA(c->tmp.ensure(ml * 16 + 2 * ml * 8));
        double* fr = reinterpret_cast<double*>(c->tmp.as<double2>() + ml);
        double* cur = fr + ml;
        FGB_CUDA(cudaMemcpyAsync(c->tmp.p, f, ml * 16, cudaMemcpyHostToDevice, c->stream));
        FGB_LAUNCH(launch_real_part(c->tmp.p, fr, (int64_t)ml, c->stream), 1);
        FGB_LAUNCH(launch_rto_tiled(fr, c->slab(1), n, c->stream), 1);
        double* prev = reinterpret_cast<double*>(c->tmp.p);  // the complex staging is free now: reuse
        if (int st = check_orthogonal(c, fr, prev)) return st;
        // Small n: one n^3 GEMM per power leaves most SMs idle (n = 1024: 64 CTA tiles), so build by
        // doubling, P_(s+j) = P_j P_s for j = 1..s: log2(L) levels of batched GEMMs over all
        // powers, same (L-1) products. The reference left-multiplies (transform.hpp:58); the
        // results agree to rounding (and the recursion depth drops from L-1 to log2 L).
        static const bool chain_only = std::getenv("FGFRFT_BUILD_CHAIN") != nullptr;
        if (!chain_only && n <= 2048 && c->l >= 4) {
            DevBuf rect;  // all L powers column-major (L n^2 doubles; <= 2 GB at n = 2048, L = 64)
            FGB_CUDA(rect.ensure(ml * 8 * (size_t)c->l));
            double* R = rect.as<double>();
            FGB_CUDA(cudaMemcpyAsync(R, fr, ml * 8, cudaMemcpyDeviceToDevice, c->stream));
            for (int s = 1; s < c->l; s *= 2) {
                const int cnt = std::min(s, c->l - s);
                ProfScope ps(KC_GEMM, c->stream);
                FGB_LAUNCH(launch_rgemm(0, 0, 0, n, n, n, R, n, (int64_t)ml, R + (size_t)(s - 1) * ml, n, 0,
                                        R + (size_t)s * ml, n, (int64_t)ml, cnt, c->stream),
                           1);
            }
            for (int k = 2; k <= c->l; ++k)
                FGB_LAUNCH(launch_rto_tiled(R + (size_t)(k - 1) * ml, c->slab(k), n, c->stream), 1);
            FGB_CUDA(cudaStreamSynchronize(c->stream));
            rect.release();
            c->tmp.release();
            return FGFRFT_OK;
        }
        // Large n: the chain P_k = F P_(k-1), on the INT8 engine with 7 digits (~1e-15 per product,
        // the DMMA rounding level) unless the engine is forced to DMMA (FGFRFT_ENGINE=dmma).
        static const bool dmma_only = [] {
            const char* e = std::getenv("FGFRFT_ENGINE");
            return e && !std::strcmp(e, "dmma");
        }();
        const bool i8 = !dmma_only && n > 2048 && n <= 16384;
        const double* p = fr;
        for (int k = 2; k <= c->l; ++k) {
            if (i8) {
                if (int st = fgfrft_dgemm_int8_dev(0, 0, n, n, n, fr, n, p, n, cur, n, 7, c->stream)) return st;
            } else {
                ProfScope ps(KC_GEMM, c->stream);
                FGB_LAUNCH(launch_rgemm(0, 0, 0, n, n, n, fr, n, 0, p, n, 0, cur, n, 0, 1, c->stream), 1);
            }
            FGB_LAUNCH(launch_rto_tiled(cur, c->slab(k), n, c->stream), 1);
            p = cur;
            std::swap(prev, cur);
        }
        FGB_CUDA(cudaStreamSynchronize(c->stream));
        c->tmp.release();
        return FGFRFT_OK;
    }
    FGB_CUDA(c->tmp.ensure(3 * ml * 16));
    double2* fbuf = c->tmp.as<double2>();
    double2* prev = fbuf + ml;
    double2* cur = fbuf + 2 * ml;
    FGB_CUDA(cudaMemcpyAsync(fbuf, f, ml * 16, cudaMemcpyHostToDevice, c->stream));
    FGB_LAUNCH(launch_to_tiled(fbuf, c->slab(1), n, (int)c->elem, c->stream), 1);
    const double2* p = fbuf;
    for (int k = 2; k <= c->l; ++k) {
        FGB_LAUNCH(launch_zgemm(n, n, n, fbuf, n, 0, false, p, n, 0, false, cur, n, 0, 1, false, c->stream), 1);
        FGB_LAUNCH(launch_to_tiled(cur, c->slab(k), n, (int)c->elem, c->stream), 1);
        p = cur;
        std::swap(prev, cur);
    }
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    c->tmp.release();
    return FGFRFT_OK;
}

int upload_powers(fgfrft_cache* c, const double* powers) {
    const size_t ml = c->mat_elems();
    FGB_CUDA(c->tmp.ensure(ml * 16 + ml * 8));
    for (int k = 1; k <= c->l; ++k) {
        FGB_CUDA(cudaMemcpyAsync(c->tmp.p, powers + 2 * ml * (k - 1), ml * 16, cudaMemcpyHostToDevice, c->stream));
        if (c->real) {
            double* fr = reinterpret_cast<double*>(c->tmp.as<double2>() + ml);
            FGB_LAUNCH(launch_real_part(c->tmp.p, fr, (int64_t)ml, c->stream), 1);
            FGB_LAUNCH(launch_rto_tiled(fr, c->slab(k), (int)c->n, c->stream), 1);
            if (k == 1)
                if (int st = check_orthogonal(c, fr, reinterpret_cast<double*>(c->tmp.p))) return st;
        } else {
            FGB_LAUNCH(launch_to_tiled(c->tmp.p, c->slab(k), (int)c->n, (int)c->elem, c->stream), 1);
        }
    }
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    c->tmp.release();
    return FGFRFT_OK;
}

// Copy n_alpha device results of the cache dtype to complex128 host matrices.
int download_as_c128(fgfrft_cache* c, const void* dev, size_t elems, double* host) {
    if (c->dtype == FGFRFT_C128) {
        FGB_CUDA(cudaMemcpyAsync(host, dev, elems * 16, cudaMemcpyDeviceToHost, c->stream));
        FGB_CUDA(cudaStreamSynchronize(c->stream));
        return FGFRFT_OK;
    }
    std::vector<float> tmp(2 * elems);
    FGB_CUDA(cudaMemcpyAsync(tmp.data(), dev, elems * 8, cudaMemcpyDeviceToHost, c->stream));
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < 2 * elems; ++i) host[i] = (double)tmp[i];
    return FGFRFT_OK;
}

int resolve_truncation(const fgfrft_cache* c, int truncation, int which, int* l_used) {
    const int l = (which == FGFRFT_DQ || truncation == 0) ? c->l : truncation;
    if (l < 1 || l > c->l) return fail(FGFRFT_PARAMETER, "fgfrft_matrix: truncation exceeds the cached power set");
    *l_used = l;
    return FGFRFT_OK;
}

int engine_of(const fgfrft_cache* c);
bool complex_int8_default(int64_t m, int64_t n, int64_t k);
int zgemm_auto(int opa, int opb, int64_t m, int64_t n, int64_t k, const void* a, int64_t lda, int64_t sa,
               const void* b, int64_t ldb, int64_t sb, void* c, int64_t ldc, int64_t sc, int batch, cudaStream_t st);

// Complex GEMM in the cache's arithmetic: complex128 on the INT8 engine (large products, engine
// not DMMA) or DMMA; FP32 for complex64.
cudaError_t gemm(const fgfrft_cache* c, int M, int N, int K, const void* A, int64_t lda, int64_t sA, bool conj_a,
                 const void* B, int64_t ldb, int64_t sB, bool conj_b, void* C, int64_t ldc, int64_t sC, int batch) {
    if (c->dtype == FGFRFT_C128 && engine_of(c) != FGFRFT_ENGINE_DMMA && complex_int8_default(M, N, K)) {
        const int r = zgemm_auto(conj_a ? 2 : 0, conj_b ? 2 : 0, M, N, K, A, lda, sA, B, ldb, sB, C, ldc, sC, batch,
                                 c->stream);
        return r == FGFRFT_OK ? cudaSuccess : cudaErrorUnknown;
    }
    if (c->dtype == FGFRFT_C128)
        return launch_zgemm(M, N, K, A, lda, sA, conj_a, B, ldb, sB, conj_b, C, ldc, sC, batch, false, c->stream);
    return launch_cgemm(M, N, K, A, lda, sA, conj_a, B, ldb, sB, conj_b, C, ldc, sC, batch, false, c->stream);
}

// Host complex128 block -> device buffer of the cache dtype (complex64: staged + demoted).
int upload_signal(fgfrft_cache* c, const double* host, size_t elems, void* dst) {
    if (c->dtype == FGFRFT_C128) {
        FGB_CUDA(cudaMemcpyAsync(dst, host, elems * 16, cudaMemcpyHostToDevice, c->stream));
        return FGFRFT_OK;
    }
    FGB_CUDA(c->tmp.ensure(elems * 16));
    FGB_CUDA(cudaMemcpyAsync(c->tmp.p, host, elems * 16, cudaMemcpyHostToDevice, c->stream));
    FGB_LAUNCH(launch_demote(c->tmp.p, dst, (int64_t)elems, c->stream), 1);
    return FGFRFT_OK;
}

// Device buffer of the cache dtype -> host complex128 (synchronises the stream).
int download_signal(fgfrft_cache* c, const void* src, size_t elems, double* host) {
    if (c->dtype == FGFRFT_C128) {
        FGB_CUDA(cudaMemcpyAsync(host, src, elems * 16, cudaMemcpyDeviceToHost, c->stream));
    } else {
        FGB_CUDA(c->tmp.ensure(elems * 16));
        FGB_LAUNCH(launch_promote(src, c->tmp.p, (int64_t)elems, c->stream), 1);
        FGB_CUDA(cudaMemcpyAsync(host, c->tmp.p, elems * 16, cudaMemcpyDeviceToHost, c->stream));
    }
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    return FGFRFT_OK;
}

// INT8 tensor-core (Ozaki) versions of the real-F synthesis route's two GEMMs (defined below).
bool use_int8_gemm(const fgfrft_cache* c, int64_t b);
bool use_fused_apply(const fgfrft_cache* c, int n_alpha, int64_t b);
int slice_signal_rows(fgfrft_cache* c, const void* x_dev, int64_t b, int64_t* bp_out, cudaStream_t st = nullptr);
int ensure_pipe_streams(fgfrft_cache* c);
int int8_gx(fgfrft_cache* c, int na, const void* g, const void* x_dev, int64_t b, void* m);
int int8_gx_gen(fgfrft_cache* c, int na, const void* g, int64_t m, const void* x_dev, int64_t b, void* out,
                int64_t sm);
bool use_power_route(const fgfrft_cache* c, int n_alpha);
int engine_of(const fgfrft_cache* c);
int apply_power_route(fgfrft_cache* c, const double* coef, int n_alpha, const void* x_dev, int64_t b, void* y_dev);
bool use_node_route(const fgfrft_cache* c, int n_alpha, int64_t b);
int mse_node_route(fgfrft_cache* c, const double* alphas, int n_alpha, const void* x_dev, const void* xc_dev,
                   int64_t b, void* y_dev, double* loss_dev, double* dlda_dev, bool need_d, bool* ran);

// Y[a] = op(Q(alpha_a)) X for all orders; x_dev n x b, y_dev n_alpha blocks of n x b.
int apply_device(fgfrft_cache* c, const double* alphas, int n_alpha, int l_used, bool inverse, const void* x_dev,
                 int64_t b, void* y_dev) {
    double* coef = nullptr;
    if (l_used == c->l && use_power_route(c, n_alpha)) {
        // Q(a)^T = Q(-a) bit-exactly (the coefficients mirror exactly, sinc.hpp / test_sinc.cpp:40-46)
        std::vector<double> al(alphas, alphas + n_alpha);
        if (inverse)
            for (double& v : al) v = -v;
        if (use_node_route(c, n_alpha, b)) {
            bool ran = false;
            if (int st = mse_node_route(c, al.data(), n_alpha, x_dev, nullptr, b, y_dev, nullptr, nullptr, false, &ran))
                return st;
            if (ran) return FGFRFT_OK;
        }
        if (int st = upload_coefs(c, al.data(), n_alpha, l_used, &coef)) return st;
        return apply_power_route(c, coef, n_alpha, x_dev, b, y_dev);
    }
    if (int st = upload_coefs(c, alphas, n_alpha, l_used, &coef)) return st;
    const int n = (int)c->n;
    const size_t sl = c->mat_elems();
    if (use_fused_apply(c, n_alpha, b)) {
        // small batch: fused synthesis + product, Q never materialised (K3)
        FGB_CUDA(c->partial.ensure(rapply_fused_part_elems(n, n_alpha) * sizeof(double)));
        const size_t width = (size_t)(2 * l_used + 1);
        std::vector<double> al(alphas, alphas + n_alpha);
        if (inverse) {  // Q(a)^T = Q(-a) bit-exactly
            for (double& v : al) v = -v;
            if (int st = upload_coefs(c, al.data(), n_alpha, l_used, &coef)) return st;
        }
        ProfScope ps(KC_SYNTH, c->stream);
        FGB_LAUNCH(launch_rapply_fused(c->slabs, n, l_used, coef, (int)width, n_alpha, static_cast<const double*>(x_dev),
                                       (int)b, c->partial.as<double>(), static_cast<double*>(y_dev), c->stream),
                   2);
        return FGFRFT_OK;
    }
    if ((n_alpha == 1 || n_alpha == 2 || n_alpha == 4) && packed_enabled(c) && use_int8_gemm(c, b)) {
        // Q(a)^T = Q(-a) bit-exactly (sinc.hpp coefficient mirror): the inverse synthesises Q(-a)
        std::vector<double> al(alphas, alphas + n_alpha);
        if (inverse)
            for (double& v : al) v = -v;
        WindowWeights ww;
        const bool win = window_weights(c, al.data(), n_alpha, false, l_used, &ww);
        if (win || ensure_step_cache(c)) {
            if (inverse)
                if (int st = upload_coefs(c, al.data(), n_alpha, l_used, &coef)) return st;
            return packed_products(c, coef, 2 * l_used + 1, n_alpha, x_dev, b, y_dev, l_used, nullptr,
                                   win ? &ww : nullptr);
        }
    }
    const int chunk = alpha_chunk(c, n_alpha);
    FGB_CUDA(c->q.ensure((size_t)chunk * sl * c->elem));
    const size_t width = (size_t)(2 * l_used + 1);
    for (int a0 = 0; a0 < n_alpha; a0 += chunk) {
        const int na = std::min(chunk, n_alpha - a0);
        if (int st = synth_into(c, coef + a0 * width, na, l_used, c->q.p, true)) return st;
        if (use_int8_gemm(c, b)) {
            if (int st = int8_qx(c, na, inverse, c->q.p, x_dev, b,
                                 static_cast<char*>(y_dev) + (size_t)a0 * n * b * c->sig))
                return st;
            continue;
        }
        ProfScope ps(KC_GEMM, c->stream);
        if (c->real)  // Y = Q X or Q^T X with real Q: real DMMA GEMM over the (re, im) columns
            FGB_LAUNCH(launch_rgemm(inverse ? 1 : 0, 1, 1, n, 2 * (int)b, n, c->q.p, n, (int64_t)sl, x_dev, n, 0,
                                    static_cast<char*>(y_dev) + (size_t)a0 * n * b * c->sig, n, (int64_t)2 * n * b, na,
                                    c->stream),
                       1);
        else
            FGB_LAUNCH(gemm(c, n, (int)b, n, c->q.p, n, (int64_t)sl, inverse, x_dev, n, 0, false,
                            static_cast<char*>(y_dev) + (size_t)a0 * n * b * c->sig, n, (int64_t)n * b, na),
                       1);
    }
    return FGFRFT_OK;
}

// ------------------------------------------------------------------ power-product route
//
// For an order sweep over a real cache, F^a X = sum_k c_k(a) F^k X: the 2L products
// Z_k = P_k X, W_k = P_k^T X are ONE INT8 tensor-core GEMM of the stacked sliced cache with X,
// after which each order is a (2L+1)-term combination (combine.cu). Used when it is cheaper than
// synthesising every Q(a): 2L products against 2 GEMMs (Q X and G X^H) per order.
int engine_of(const fgfrft_cache* c) {
    if (c->engine != FGFRFT_ENGINE_AUTO) return c->engine;
    static const int env = [] {
        const char* e = std::getenv("FGFRFT_ENGINE");
        if (!e) return (int)FGFRFT_ENGINE_AUTO;
        if (!std::strcmp(e, "dmma")) return (int)FGFRFT_ENGINE_DMMA;
        if (!std::strcmp(e, "int8")) return (int)FGFRFT_ENGINE_INT8;
        return (int)FGFRFT_ENGINE_AUTO;
    }();
    return env;
}

int64_t pad_rows(int64_t n) { return ceil_div(n, kOzTileA) * kOzTileA; }
int64_t pad_k(int64_t n) { return ceil_div(n, kOzK) * kOzK; }

// Device bytes of the INT8 digit slices the sweep routes build once per cache (counted against
// the handle's memory budget, aux_fits): the stacked cache for the power route, its element rows
// for the node route.
uint64_t power_slice_bytes(const fgfrft_cache* c) {
    const uint64_t rows = 2 * (uint64_t)c->l * pad_rows(c->n);
    return (uint64_t)oz_slices_default() * rows * pad_k(c->n) + rows * 12;
}
// The node operators' A operand: element-PAIR rows by default (row = the element pair (i, j), (j, i)
// of a tile pair, K = the L powers of both elements: half the bytes of the element-row form, whose
// K stacked P_k(i, j) and P_k(j, i) for every element, so every power was stored twice) -- the
// same values per row, so the same slicing error. Measured at config 2 it reads half the bytes (427
// vs 812 MB, ncu) but runs slower: 0.217 ms (vs 0.182) with the 64-column B tile (its 6 digit-sum
// accumulators, 384 TMEM columns, leave room for ONE buffer: every unit's MMAs wait for the previous
// unit's epilogue) and 0.30 ms as two double-buffered 32-column units per tile -- half of every
// pair's outputs are the mirror elements, whose column-major stores scatter one 8-byte word per lane
// (the pair's mirror rows come from 8 different units, too many to transpose through shared
// memory). Opt-in (FGFRFT_NODE_PAIRS=1).
static bool node_pairs_wanted() {
    static const bool v = [] {
        const char* e = std::getenv("FGFRFT_NODE_PAIRS");
        return e && std::atoi(e) == 1;
    }();
    return v;
}

uint64_t elem_slice_bytes(const fgfrft_cache* c) {
    if (node_pairs_wanted()) {
        const uint64_t rows = dsynth_cache_rows((int)c->n);
        return (uint64_t)oz_slices_default() * rows * dsynth_kp(c->l) + rows * 12;
    }
    const uint64_t rows = pad_rows(c->n * c->n);
    return (uint64_t)oz_slices_default() * rows * pad_k(2 * (int64_t)c->l) + rows * 12;
}

static bool power_route_shape(const fgfrft_cache* c, int n_alpha) {
    if (!c->real || c->dtype != FGFRFT_C128 || 2 * c->l + 1 > combine_max_terms() || c->n > 16384) return false;
    const int eng = engine_of(c);
    if (eng == FGFRFT_ENGINE_DMMA) return false;
    if (eng == FGFRFT_ENGINE_INT8 || eng == FGFRFT_ENGINE_INT8_COMBINE) return true;
    return 2 * n_alpha >= c->l;  // auto: 2L products amortised over the orders
}

bool use_power_route(const fgfrft_cache* c, int n_alpha) {
    return power_route_shape(c, n_alpha) && (c->ps_slices || aux_fits(c, power_slice_bytes(c)));
}

int wait_xc(fgfrft_cache* c);

// ------------------------------------------------------------------ node route
//
// For an order sweep on [lo, hi], Q(a) = sum_k c_k(a) P_k is an entire function of a, so it is
// interpolated to rounding by a degree-(r-1) polynomial through r Chebyshev nodes a_j of the
// interval (r = 19 for a width-2 sweep: 4e-15 on the coefficients, 2e-12 on their derivatives,
// checked per call): F^a X = sum_j l_j(a) W_j X and dF^a/da X = sum_j l_j'(a) W_j X with the node
// operators W_j = Q(a_j). The W_j come from ONE INT8 GEMM over the cache's 2L terms (element-row
// digit slices of the stacked cache x the node coefficient rows), the products W_j X from a
// second one, and the per-order Y, dY, loss and dL/da from one DMMA pass over the r products
// (node_combine_kernel) -- r products instead of the power route's 2L. Every call re-plans
// (memoised on the order set): nodes, barycentric weights, an interpolation check against the
// exact coefficients of every order; no r <= 48 passing the check falls back to the power route.
bool use_node_route(const fgfrft_cache* c, int n_alpha, int64_t b) {
    static const int mode = [] {
        const char* e = std::getenv("FGFRFT_ROUTE");
        return (e && !std::strcmp(e, "power")) ? 0 : 1;
    }();
    return mode == 1 && power_route_shape(c, n_alpha) && engine_of(c) == FGFRFT_ENGINE_AUTO && use_int8_gemm(c, b) &&
           n_alpha >= 16 && n_alpha <= 64 && c->n <= 46340 && (c->es_slices || aux_fits(c, elem_slice_bytes(c)));
}

int ensure_elem_slices(fgfrft_cache* c) {
    const int S = oz_slices_default();
    if (c->es_slices == S) return FGFRFT_OK;
    if (node_pairs_wanted()) {
        const int64_t rows = (int64_t)dsynth_cache_rows((int)c->n), kp = dsynth_kp(c->l);
        FGB_CUDA(c->es.ensure((size_t)S * rows * kp));
        FGB_CUDA(c->ee.ensure((size_t)rows * sizeof(int)));
        FGB_CUDA(c->erm.ensure((size_t)rows * sizeof(unsigned long long)));
        ProfScope ps(KC_SLICE, c->stream);
        FGB_LAUNCH(launch_dsynth_build(static_cast<const double*>(c->slabs), (int)c->n, c->l, (int)kp,
                                       c->es.as<int8_t>(), c->ee.as<int>(), c->erm.as<unsigned long long>(), c->stream,
                                       S),
                   3);
        c->es_slices = S;
        c->es_pairs = true;
        c->aux_bytes += elem_slice_bytes(c);
        return FGFRFT_OK;
    }
    const int64_t n = c->n, rows = pad_rows(n * n), kp = pad_k(2 * (int64_t)c->l);
    FGB_CUDA(c->es.ensure((size_t)S * rows * kp));
    FGB_CUDA(c->ee.ensure((size_t)rows * sizeof(int)));
    FGB_CUDA(c->erm.ensure((size_t)rows * sizeof(unsigned long long)));
    OzView v{static_cast<const double*>(c->slabs), 0, 0, (int64_t)c->slab_elems(), 0, 0, (int)(n * n), (int)rows, 1,
             2 * c->l, (int)kp, true};
    v.tiled = 6;
    v.nt = (int)ceil_div(n, kTile);
    v.l = c->l;
    v.tp2 = (int)n;
    ProfScope ps(KC_SLICE, c->stream);
    FGB_LAUNCH(launch_oz_slice(v, S, kOzTileA, c->es.as<int8_t>(), c->ee.as<int>(), c->erm.as<unsigned long long>(),
                               c->stream),
               3);
    c->es_slices = S;
    c->aux_bytes += elem_slice_bytes(c);
    return FGFRFT_OK;
}

// Plan: nodes, node coefficient rows (r x T), interpolation weights P = [l_j(a); l_j'(a)] (rows x rp).
// coef_h holds the exact [c | c'] tables of the orders (upload_coefs). The node count is the
// smallest r (from an estimate upward) whose interpolated coefficients match the exact ones on
// every order to 4e-15 of the largest coefficient (2e-12 for the derivatives) -- about 9 + 5w for
// a width-w sweep (19 for [0, 2]). false: not interpolable within node_max_terms() nodes.
static bool node_plan_r(const double* alphas, int na, int l, bool need_d, const double* coef_h, int r,
                        std::vector<double>& tab, std::vector<double>& d0, std::vector<double>& pw, int* rp_out) {
    const int T = 2 * l + 1;
    double lo = alphas[0], hi = alphas[0];
    for (int a = 1; a < na; ++a) {
        lo = std::min(lo, alphas[a]);
        hi = std::max(hi, alphas[a]);
    }
    const double w = hi - lo;
    const int rp = (r + 3) / 4 * 4;
    const double mid = 0.5 * (lo + hi), half = 0.5 * w;
    std::vector<double> xn((size_t)r), bw((size_t)r);
    for (int j = 0; j < r; ++j) {  // Chebyshev points of the first kind and their barycentric weights
        const double th = M_PI * (2.0 * j + 1.0) / (2.0 * r);
        xn[j] = mid + half * std::cos(th);
        bw[j] = ((j & 1) ? -1.0 : 1.0) * std::sin(th);
    }
    tab.assign((size_t)r * T, 0.0);
    d0.assign((size_t)r, 0.0);
    std::vector<double> scratch((size_t)T);
    for (int j = 0; j < r; ++j) {
        host_sinc_coeffs_fast(xn[j], l, &tab[(size_t)j * T], scratch.data());
        d0[j] = tab[(size_t)j * T + l];
    }
    const int rows = need_d ? 2 * na : na;
    pw.assign((size_t)rows * rp, 0.0);
    for (int a = 0; a < na; ++a) {
        const double x = alphas[a];
        double* lj = &pw[(size_t)a * rp];
        double* dj = need_d ? &pw[(size_t)(na + a) * rp] : nullptr;
        int hit = -1;
        for (int j = 0; j < r; ++j)
            if (std::fabs(x - xn[j]) < 1e-14 * std::max(1.0, std::fabs(x))) hit = j;
        if (hit >= 0) {  // on a node: Kronecker weights, the derivative row of the differentiation matrix
            lj[hit] = 1.0;
            if (dj) {
                double diag = 0.0;
                for (int j = 0; j < r; ++j)
                    if (j != hit) {
                        dj[j] = (bw[j] / bw[hit]) / (xn[hit] - xn[j]);
                        diag -= dj[j];
                    }
                dj[hit] = diag;
            }
            continue;
        }
        double sw = 0.0, sw2 = 0.0;
        for (int j = 0; j < r; ++j) {
            const double t = bw[j] / (x - xn[j]);
            sw += t;
            sw2 += t / (x - xn[j]);
        }
        for (int j = 0; j < r; ++j) {
            const double t = bw[j] / (x - xn[j]);
            lj[j] = t / sw;
            if (dj) dj[j] = lj[j] * (-1.0 / (x - xn[j]) + sw2 / sw);
        }
    }
    *rp_out = rp;
    // The derivative weights l_j'(a) amplify the node operators' INT8 error (~5e-14 of |W_j|) by
    // sum_j |l_j'(a)| ~ 420 / width: capped at 5000 (width >~ 0.08; the parity tests hold 1e-10 at
    // width 0.1) -- narrower sweeps take the power route (2L products, no derivative amplification).
    if (need_d)
        for (int a = 0; a < na; ++a) {
            double t = 0.0;
            for (int j = 0; j < r; ++j) t += std::fabs(pw[(size_t)(na + a) * rp + j]);
            if (t > 5000.0) return false;
        }
    // check the interpolated coefficients against the exact ones on every order, leaving at the
    // first miss (the search tries node counts upward: only the accepted count runs the whole check)
    double cmax = 0.0, dmax = 0.0;
    for (int a = 0; a < na; ++a)
        for (int q = 0; q < T; ++q) {
            cmax = std::max(cmax, std::fabs(coef_h[(size_t)a * T + q]));
            if (need_d) dmax = std::max(dmax, std::fabs(coef_h[(size_t)(na + a) * T + q]));
        }
    const double ctol = 4e-15 * cmax, dtol = 2e-12 * std::max(dmax, 1e-300);
    std::vector<double> vc((size_t)T), vd((size_t)T);
    double* __restrict__ pc = vc.data();
    double* __restrict__ pd = vd.data();
    for (int a = 0; a < na; ++a) {
        const double* c = coef_h + (size_t)a * T;
        const double* dc = coef_h + (size_t)(na + a) * T;
        std::fill(vc.begin(), vc.end(), 0.0);
        std::fill(vd.begin(), vd.end(), 0.0);
        for (int j = 0; j < r; ++j) {
            const double* __restrict__ tj = &tab[(size_t)j * T];
            const double pl = pw[(size_t)a * rp + j], pdj = need_d ? pw[(size_t)(na + a) * rp + j] : 0.0;
            for (int q = 0; q < T; ++q) {
                pc[q] += pl * tj[q];
                pd[q] += pdj * tj[q];
            }
        }
        for (int q = 0; q < T; ++q) {
            if (std::fabs(pc[q] - c[q]) > ctol) return false;
            if (need_d && std::fabs(pd[q] - dc[q]) > dtol) return false;
        }
    }
    return true;
}

bool node_plan(fgfrft_cache* c, const double* alphas, int na, bool need_d, int* r_out, int* rp_out) {
    auto& p = c->nd_plan;
    if (p.need_d == need_d && p.alphas.size() == (size_t)na &&
        !std::memcmp(p.alphas.data(), alphas, (size_t)na * sizeof(double))) {
        *r_out = p.r;
        *rp_out = p.rp;
        return p.ok;
    }
    p.alphas.assign(alphas, alphas + na);
    p.need_d = need_d;
    p.ok = false;
    p.staged = false;
    double lo = alphas[0], hi = alphas[0];
    for (int a = 1; a < na; ++a) {
        lo = std::min(lo, alphas[a]);
        hi = std::max(hi, alphas[a]);
    }
    const double w = hi - lo;
    if (!(w > 1e-9)) return false;
    // the element-pair node operators hold 2r <= 64 output columns (one B tile)
    const int rmax = node_pairs_wanted() ? std::min(node_max_terms(), kOzTileB / 2) : node_max_terms();
    // the orders' exact coefficient tables for the interpolation check (host only)
    const int T = 2 * c->l + 1;
    c->nd_ctab.resize((size_t)2 * na * T);
    for (int a = 0; a < na; ++a)
        host_sinc_coeffs_fast(alphas[a], c->l, &c->nd_ctab[(size_t)a * T], &c->nd_ctab[(size_t)(na + a) * T]);
    // the search starts one below the count the last sweep of (almost) the same width needed -- the
    // counts below it fail their first orders cheaply, but each still costs its node table
    int r0 = std::max(6, (int)std::floor(8.0 + 4.2 * w));
    if (p.hint_r > 0 && p.hint_need_d == need_d && std::fabs(p.hint_w - w) <= 1e-6 * w) r0 = std::max(r0, p.hint_r - 1);
    for (int r = r0; r <= rmax; ++r)
        if (node_plan_r(alphas, na, c->l, need_d, c->nd_ctab.data(), r, p.tab, p.d0, p.pw, &p.rp)) {
            p.r = r;
            p.ok = true;
            p.hint_r = r;
            p.hint_w = w;
            p.hint_need_d = need_d;
            break;
        }
    *r_out = p.r;
    *rp_out = p.rp;
    return p.ok;
}

// The element-pair form of node_products: one INT8 GEMM over the pair-major slices (L terms per
// element instead of 2L) with 2r output columns (W_j at the pair's element and at its mirror),
// the diagonal and the row maxima of W fused into the epilogue (ozgemm pair mode).
static int node_products_pairs(fgfrft_cache* c, const std::vector<double>& tab, const std::vector<double>& d0, int r,
                               const void* x_dev, int64_t b, bool upload) {
    const int S = c->es_slices;
    // B: 2r rows sliced as two 32-row tiles (64 rows: the slicer's granule); the narrow,
    // double-buffered GEMM form runs over the live tiles
    const int64_t n = c->n, rows = (int64_t)dsynth_cache_rows((int)n), kp = dsynth_kp(c->l), bp = kOzTileB;
    const int64_t bn = ceil_div(2 * r, kOzTileNarrow) * kOzTileNarrow;
    if (upload) {
        FGB_CUDA(c->nd_tab.ensure(tab.size() * 8));
        FGB_CUDA(c->nd_d0.ensure(d0.size() * 8));
        FGB_CUDA(cudaMemcpyAsync(c->nd_tab.p, c->nd_h, tab.size() * 8, cudaMemcpyHostToDevice, c->stream));
        FGB_CUDA(cudaMemcpyAsync(c->nd_d0.p, c->nd_h + tab.size(), d0.size() * 8, cudaMemcpyHostToDevice, c->stream));
    }
    FGB_CUDA(c->nd_bsl.ensure((size_t)S * bp * kp));
    FGB_CUDA(c->nd_bex.ensure((size_t)bp * (sizeof(int) + sizeof(unsigned long long))));
    int* be = c->nd_bex.as<int>();
    {  // B rows 2x + m: node x's coefficients in the pair order (OzView mode 8)
        OzView v{c->nd_tab.as<double>(), 2 * c->l + 1, 0, 0, 0, 0, 2 * r, (int)bp, 1, (int)kp, (int)kp, false};
        v.tiled = 8;
        v.l = c->l;
        ProfScope ps(KC_SLICE, c->stream);
        FGB_LAUNCH(launch_oz_slice(v, S, kOzTileNarrow, c->nd_bsl.as<int8_t>(), be,
                                   reinterpret_cast<unsigned long long*>(be + bp), c->stream),
                   3);
    }
    const size_t nn = (size_t)n * n;
    FGB_CUDA(c->nd_w.ensure((size_t)r * nn * 8));
    FGB_CUDA(c->nd_z.ensure((size_t)r * n * b * 16));
    const int64_t wrows = (int64_t)r * pad_rows(n);
    FGB_CUDA(c->qsl.ensure((size_t)S * wrows * pad_k(n)));
    FGB_CUDA(c->qex.ensure((size_t)wrows * (sizeof(int) + sizeof(unsigned long long))));
    FGB_CUDA(cudaMemsetAsync(c->qex.as<int>() + wrows, 0, (size_t)wrows * sizeof(unsigned long long), c->stream));
    {
        OzOut out;
        out.c = c->nd_w.as<double>();
        out.ldc = (int64_t)nn;
        out.sc = 0;
        out.mv = (int)rows;
        out.mp = (int)rows;
        out.nv = 2 * r;
        out.rmax = reinterpret_cast<unsigned long long*>(c->qex.as<int>() + wrows);
        out.dg = c->nd_d0.as<double>();
        out.rnp = (int)pad_rows(n);
        out.pair_nt = (int)ceil_div(n, kTile);
        out.pair_n = (int)n;
        ProfScope ps(KC_NODEOP, c->stream);
        FGB_LAUNCH(launch_ozgemm_narrow(S, c->es.as<int8_t>(), c->ee.as<int>(), (int)rows, c->nd_bsl.as<int8_t>(), be,
                                        (int)bn, (int)kp, out, c->stream),
                   1);
    }
    return int8_qx(c, r, false, c->nd_w.p, x_dev, b, c->nd_z.p, true);
}

// W_j = sum_k c_k(a_j) P_k (INT8 GEMM over the element-row slices) and Z'_j = W_j X.
int node_products(fgfrft_cache* c, const std::vector<double>& tab, const std::vector<double>& d0, int r,
                  const void* x_dev, int64_t b, bool upload) {
    if (int st = ensure_elem_slices(c)) return st;
    const int S = c->es_slices;
    const int T = 2 * c->l + 1;
    if (c->es_pairs) {
        if (r > kOzTileB / 2) return fail(FGFRFT_NUMERICAL, "node route: more nodes than the pair form holds");
        return node_products_pairs(c, tab, d0, r, x_dev, b, upload);
    }
    const int64_t n = c->n, rows = pad_rows(n * n), kp = pad_k(2 * (int64_t)c->l), bp = kOzTileB;
    // X's digits (the product GEMM's B operand) on the side stream, beside the node-operator GEMM
    // (ordered after everything already on c->stream: the previous call's product GEMM read them)
    static const bool x_side = [] {
        const char* e = std::getenv("FGFRFT_NODE_XSIDE");
        return !e || std::atoi(e) != 0;
    }();
    int64_t xbp = 0;
    cudaEvent_t xev = nullptr;
    if (x_side) {
        if (int st = ensure_pipe_streams(c)) return st;
        FGB_CUDA(cudaEventRecord(c->pk_e0, c->stream));
        FGB_CUDA(cudaStreamWaitEvent(c->pk_g, c->pk_e0, 0));
        if (int st = slice_signal_rows(c, x_dev, b, &xbp, c->pk_g)) return st;
        FGB_CUDA(cudaEventRecord(c->pk_ex, c->pk_g));
        xev = c->pk_ex;
    }
    // The node tables come from the host plan, not from the stream's earlier work: their upload and
    // slicing run on the second side stream, ordered only after the previous call's node-operator
    // GEMM (the reader of these buffers), so in back-to-back steps they overlap the previous step's tail.
    cudaStream_t ts = x_side ? c->pk_s : c->stream;
    if (x_side && c->nd_ev_op) FGB_CUDA(cudaStreamWaitEvent(ts, c->nd_ev_op, 0));
    FGB_CUDA(c->nd_tab.ensure(tab.size() * 8));
    FGB_CUDA(c->nd_d0.ensure(d0.size() * 8));
    if (upload) {
        FGB_CUDA(cudaMemcpyAsync(c->nd_tab.p, c->nd_h, tab.size() * 8, cudaMemcpyHostToDevice, ts));
        FGB_CUDA(cudaMemcpyAsync(c->nd_d0.p, c->nd_h + tab.size(), d0.size() * 8, cudaMemcpyHostToDevice, ts));
    }
    FGB_CUDA(c->nd_bsl.ensure((size_t)S * bp * kp));
    FGB_CUDA(c->nd_bex.ensure((size_t)bp * (sizeof(int) + sizeof(unsigned long long))));
    int* be = c->nd_bex.as<int>();
    // r <= 32 nodes: the narrow GEMM form (32-row B tiles, double-buffered TMEM accumulators)
    const bool narrow = r <= kOzTileNarrow;
    {  // node coefficient rows in the stacked term order (operand mode 4)
        OzView v{c->nd_tab.as<double>(), T, 0, 0, 0, 0, r, (int)bp, 1, 2 * c->l, (int)kp, false};
        v.tiled = 4;
        v.l = c->l;
        ProfScope ps(KC_SLICE, ts);
        FGB_LAUNCH(launch_oz_slice(v, S, narrow ? kOzTileNarrow : kOzTileB, c->nd_bsl.as<int8_t>(), be,
                                   reinterpret_cast<unsigned long long*>(be + bp), ts),
                   3);
    }
    if (x_side) {
        if (!c->nd_ev_b) FGB_CUDA(cudaEventCreateWithFlags(&c->nd_ev_b, cudaEventDisableTiming));
        FGB_CUDA(cudaEventRecord(c->nd_ev_b, ts));
        FGB_CUDA(cudaStreamWaitEvent(c->stream, c->nd_ev_b, 0));
    }
    const size_t nn = (size_t)n * n;
    FGB_CUDA(c->nd_w.ensure((size_t)r * nn * 8));
    FGB_CUDA(c->nd_z.ensure((size_t)r * n * b * 16));
    // n % 128 == 0: the node-operator GEMM also adds the diagonal and leaves the row maxima of W
    // for the product GEMM's slicing (one pass over W instead of two)
    // (the GEMM's grid becomes a multiple of the n / 128 row blocks: only when that keeps >= 90% of
    // the SMs)
    const int64_t ibs = n / kOzTileA;
    static const bool fuse_ok = [] {
        const char* e = std::getenv("FGFRFT_NODE_FUSED_ROWMAX");
        return !e || std::atoi(e) != 0;
    }();
    // (only the narrow, r <= 32, epilogue implements the fusion)
    const bool fused = fuse_ok && narrow && n % kOzTileA == 0 && rows == (int64_t)nn &&
                       (FGFRFT_SMS / ibs) * ibs * 10 >= FGFRFT_SMS * 9;
    const int64_t wrows = (int64_t)r * pad_rows(n);
    if (fused) {
        FGB_CUDA(c->qsl.ensure((size_t)S * wrows * pad_k(n)));
        FGB_CUDA(c->qex.ensure((size_t)wrows * (sizeof(int) + sizeof(unsigned long long))));
        FGB_CUDA(cudaMemsetAsync(c->qex.as<int>() + wrows, 0, (size_t)wrows * sizeof(unsigned long long), c->stream));
    }
    {
        OzOut out;
        out.c = c->nd_w.as<double>();
        out.ldc = (int64_t)nn;
        out.sc = 0;
        out.mv = (int)nn;
        out.mp = (int)rows;
        out.nv = r;
        if (fused) {
            out.rmax = reinterpret_cast<unsigned long long*>(c->qex.as<int>() + wrows);
            out.dg = c->nd_d0.as<double>();
            out.rn = (int)n;
            out.rnp = (int)pad_rows(n);
        }
        ProfScope ps(KC_NODEOP, c->stream);
        if (narrow)
            FGB_LAUNCH(launch_ozgemm_narrow(S, c->es.as<int8_t>(), c->ee.as<int>(), (int)rows, c->nd_bsl.as<int8_t>(),
                                            be, kOzTileNarrow, (int)kp, out, c->stream),
                       1);
        else
            FGB_LAUNCH(launch_ozgemm_ex(S, 0, c->es.as<int8_t>(), c->ee.as<int>(), (int)rows, c->nd_bsl.as<int8_t>(),
                                        be, (int)bp, (int)kp, out, c->stream),
                       1);
    }
    if (!fused)
        FGB_LAUNCH(launch_add_diag(c->nd_w.as<double>(), (int)n, (int64_t)nn, c->nd_d0.as<double>(), r, c->stream), 1);
    if (x_side) {  // the coefficient digits and the diagonal have been read
        if (!c->nd_ev_op) FGB_CUDA(cudaEventCreateWithFlags(&c->nd_ev_op, cudaEventDisableTiming));
        FGB_CUDA(cudaEventRecord(c->nd_ev_op, c->stream));
    }
    return int8_qx(c, r, false, c->nd_w.p, x_dev, b, c->nd_z.p, fused, xev, xbp);
}

// Copy the plan's tables into the next pinned staging slot (after the uploads of the call that
// last used it, kNdRing calls ago, have read it) and upload the interpolation weights;
// node_products uploads the rest from the same slot.
int node_stage(fgfrft_cache* c, const std::vector<double>& tab, const std::vector<double>& d0,
               const std::vector<double>& pw) {
    const size_t need = tab.size() + d0.size() + pw.size();
    const int q = (c->nd_slot + 1) % fgfrft_cache::kNdRing;
    if (c->nd_evr[q]) FGB_CUDA(cudaEventSynchronize(c->nd_evr[q]));
    if (c->nd_hr_cap[q] < need) {
        if (c->nd_hr[q]) cudaFreeHost(c->nd_hr[q]);
        c->nd_hr[q] = nullptr;
        c->nd_hr_cap[q] = 0;
        FGB_CUDA(cudaMallocHost(&c->nd_hr[q], need * 8));
        c->nd_hr_cap[q] = need;
    }
    c->nd_slot = q;
    c->nd_h = c->nd_hr[q];
    std::memcpy(c->nd_h, tab.data(), tab.size() * 8);
    std::memcpy(c->nd_h + tab.size(), d0.data(), d0.size() * 8);
    std::memcpy(c->nd_h + tab.size() + d0.size(), pw.data(), pw.size() * 8);
    FGB_CUDA(c->nd_p.ensure(pw.size() * 8));
    FGB_CUDA(cudaMemcpyAsync(c->nd_p.p, c->nd_h + tab.size() + d0.size(), pw.size() * 8, cudaMemcpyHostToDevice,
                             c->stream));
    return FGFRFT_OK;
}

// record that the staging may be reused once the uploads enqueued so far have run
int node_staged(fgfrft_cache* c) {
    cudaEvent_t& ev = c->nd_evr[c->nd_slot];
    if (!ev) FGB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    FGB_CUDA(cudaEventRecord(ev, c->stream));
    return FGFRFT_OK;
}

// Y (optional), loss, dL/da of an order sweep through the node route; false in *ran when the
// sweep is not interpolable (the caller falls back).
int mse_node_route(fgfrft_cache* c, const double* alphas, int n_alpha, const void* x_dev, const void* xc_dev,
                   int64_t b, void* y_dev, double* loss_dev, double* dlda_dev, bool need_d, bool* ran) {
    *ran = false;
    int r = 0, rp = 0;
    {
        HostTimer ht(1);
        if (!node_plan(c, alphas, n_alpha, need_d, &r, &rp)) return FGFRFT_OK;
    }
    auto& p = c->nd_plan;
    // a memoised plan's tables are still on the device from the call that staged them: no host
    // staging, no wait on that call's uploads
    const bool upload = !p.staged;
    if (upload) {
        HostTimer ht(2);
        if (int st = node_stage(c, p.tab, p.d0, p.pw)) return st;
    }
    {
        HostTimer ht(3);
        if (int st = node_products(c, p.tab, p.d0, r, x_dev, b, upload)) return st;
    }
    if (upload) {
        if (int st = node_staged(c)) return st;
        p.staged = true;
    }
    if (xc_dev && !need_d) return fail(FGFRFT_PARAMETER, "node route: the MSE form needs the derivative rows");
    if (xc_dev)
        if (int st = wait_xc(c)) return st;
    FGB_CUDA(c->partial.ensure(node_partial_elems() * sizeof(double)));
    ProfScope ps(KC_COMBINE, c->stream);
    FGB_LAUNCH(launch_node_combine(c->nd_z.as<double>(), static_cast<const double*>(xc_dev), 2 * c->n * b, r, rp,
                                   c->nd_p.as<double>(), n_alpha, static_cast<double*>(y_dev), c->partial.as<double>(),
                                   1.0 / ((double)c->n * (double)b), loss_dev, dlda_dev, c->stream),
               xc_dev ? 2 : 1);
    // alpha = 0 exactly: Q(0) = I (sinc.hpp:16 Kronecker coefficients, test_transform.cpp:60-65), so
    // Y = X bit for bit and the loss is ||X - Xc||^2 / (N B) -- snapped instead of interpolated.
    // (Other integer orders keep the INT8 product error, <= 3e-13 relative, like every order.)
    for (int a = 0; a < n_alpha; ++a) {
        if (alphas[a] != 0.0) continue;
        const size_t blk = (size_t)2 * c->n * b;
        if (y_dev)
            FGB_CUDA(cudaMemcpyAsync(static_cast<double*>(y_dev) + (size_t)a * blk, x_dev, blk * 8,
                                     cudaMemcpyDeviceToDevice, c->stream));
        if (xc_dev && loss_dev) {
            FGB_CUDA(c->lpart.ensure((mse_dy_part_elems() + 1) * sizeof(double)));
            double* scratch = c->lpart.as<double>() + mse_dy_part_elems();  // the dot of X with itself: unused
            FGB_LAUNCH(launch_mse_dy(x_dev, x_dev, xc_dev, c->n * b, nullptr, c->lpart.as<double>(),
                                     1.0 / ((double)c->n * (double)b), loss_dev + a, scratch, c->stream),
                       2);
        }
    }
    *ran = true;
    c->last_route = 2;
    c->last_nodes = r;
    return FGFRFT_OK;
}

int ensure_power_slices(fgfrft_cache* c) {
    const int S = oz_slices_default();
    if (c->ps_slices == S) return FGFRFT_OK;
    const int64_t n = c->n, np = pad_rows(n), kp = pad_k(n), rows = 2 * (int64_t)c->l * np;
    FGB_CUDA(c->ps.ensure((size_t)S * rows * kp));
    FGB_CUDA(c->pe.ensure((size_t)rows * sizeof(int)));
    FGB_CUDA(c->prm.ensure((size_t)rows * sizeof(unsigned long long)));
    const int nt = (int)ceil_div(n, kTile);
    for (int half = 0; half < 2; ++half) {
        OzView v{static_cast<const double*>(c->slabs), 0, 0, (int64_t)c->slab_elems(), 0, 0, (int)n, (int)np, c->l,
                 (int)n, (int)kp, half == 0};
        v.tiled = half == 0 ? 1 : 2;
        v.nt = nt;
        const int64_t r0 = half * (int64_t)c->l * np;
        ProfScope ps(KC_SLICE, c->stream);
        FGB_LAUNCH(launch_oz_slice(v, S, kOzTileA, c->ps.as<int8_t>() + (size_t)S * r0 * kp, c->pe.as<int>() + r0,
                                   c->prm.as<unsigned long long>(), c->stream),
                   3);
    }
    c->ps_slices = S;
    c->aux_bytes += power_slice_bytes(c);
    return FGFRFT_OK;
}

// z <- [P_1 X; ..; P_L X; P_1^T X; ..; P_L^T X], 2L blocks of n x b complex (column-major).
int power_products(fgfrft_cache* c, const void* x_dev, int64_t b) {
    if (int st = ensure_power_slices(c)) return st;
    const int S = c->ps_slices;
    const int64_t n = c->n, np = pad_rows(n), kp = pad_k(n), rows = 2 * (int64_t)c->l * np;
    const int64_t bp = ceil_div(2 * b, kOzTileB) * kOzTileB;
    FGB_CUDA(c->xsl.ensure((size_t)S * bp * kp));
    FGB_CUDA(c->xex.ensure((size_t)bp * (sizeof(int) + sizeof(unsigned long long))));
    FGB_CUDA(c->z.ensure((size_t)2 * c->l * n * b * 16));
    int* xe = c->xex.as<int>();
    unsigned long long* xr = reinterpret_cast<unsigned long long*>(xe + bp);
    {
        // B operand rows r = 2j + comp (column j of X, re / im), K = signal index i
        const OzView v{static_cast<const double*>(x_dev), 2 * n, 2, 0, 1, 0, (int)(2 * b), (int)bp, 1, (int)n,
                       (int)kp, false};
        ProfScope ps(KC_SLICE, c->stream);
        FGB_LAUNCH(launch_oz_slice(v, S, kOzTileB, c->xsl.as<int8_t>(), xe, xr, c->stream), 3);
    }
    ProfScope ps(KC_I8GEMM, c->stream);
    FGB_LAUNCH(launch_ozgemm(S, 1, c->ps.as<int8_t>(), c->pe.as<int>(), (int)rows, c->xsl.as<int8_t>(), xe, (int)bp,
                             (int)kp, c->z.as<double>(), n, 2 * n * b, (int)n, (int)np, (int)(2 * b), c->stream),
               1);
    return FGFRFT_OK;
}

int wait_xc(fgfrft_cache* c) {
    if (!c->xc_pending) return FGFRFT_OK;
    c->xc_pending = false;
    FGB_CUDA(cudaStreamWaitEvent(c->stream, c->xc_evt, 0));
    return FGFRFT_OK;
}

bool gram_route(const fgfrft_cache* c) {
    static const bool off = std::getenv("FGFRFT_NO_GRAM") != nullptr;
    return c->orthogonal && !off;
}

// ---- INT8 combination (orthogonal F, 32 <= L <= 64): Z = F^k X never exists in FP64. The
// Z GEMM epilogue writes base-254 digits of Z (2^e_j > |x_j| >= |Z_k[i, j]|) straight into the
// A-operand layout of the combine GEMM Y = C Z, and accumulates <X, Z_k>, <Xc, Z_k>, <Z_L, Z_k>
// for the Gram form of s_k; the combine GEMM adds c_0 X, stores Y if asked and sums the loss.
int tp2_of(const fgfrft_cache* c) { return 2 * c->l <= 64 ? 64 : 128; }

// Opt-in (FGFRFT_ENGINE_INT8_COMBINE): measured on B200 it does not beat the DMMA combination at
// K = 2L = 128 -- the digit fold of the Ozaki epilogue (~60 instructions per output) outweighs
// the 2L-deep int8 products; it pays off only for much longer series.
bool use_int8_combine(const fgfrft_cache* c) {
    return engine_of(c) == FGFRFT_ENGINE_INT8_COMBINE && gram_route(c) && c->l >= 32 && c->l <= 64 &&
           c->n % 64 == 0;
}

int ensure_power_slices3(fgfrft_cache* c) {
    const int S = oz_slices_default();
    if (c->ps3_slices == S) return FGFRFT_OK;
    const int64_t n = c->n, kp = pad_k(n), tp2 = tp2_of(c);
    const int64_t rows = ceil_div(n * tp2, kOzTileA) * kOzTileA;
    FGB_CUDA(c->ps3.ensure((size_t)S * rows * kp));
    FGB_CUDA(c->pe3.ensure((size_t)rows * sizeof(int)));
    FGB_CUDA(c->prm.ensure((size_t)std::max<int64_t>(rows, 2 * c->l * pad_rows(n)) * sizeof(unsigned long long)));
    OzView v{static_cast<const double*>(c->slabs), 0, 0, (int64_t)c->slab_elems(), 0, 0, (int)n, (int)rows, 1,
             (int)n, (int)kp, false};
    v.tiled = 3;
    v.nt = (int)ceil_div(n, kTile);
    v.l = c->l;
    v.tp2 = (int)tp2;
    {
        ProfScope ps(KC_SLICE, c->stream);
        FGB_LAUNCH(launch_oz_slice(v, S, kOzTileA, c->ps3.as<int8_t>(), c->pe3.as<int>(),
                                   c->prm.as<unsigned long long>(), c->stream),
                   3);
    }
    c->ps3_slices = S;
    return FGFRFT_OK;
}

int mse_int8_combine(fgfrft_cache* c, const double* coef, const double* dcoef, int n_alpha, const void* x_dev,
                     const void* xc_dev, int64_t b, void* y_dev, double* loss_dev, double* s_dev, double* dlda_dev) {
    if (int st = ensure_power_slices3(c)) return st;
    const int S = c->ps3_slices, l = c->l, T = 2 * l + 1;
    const int64_t n = c->n, kp = pad_k(n), tp2 = tp2_of(c);
    const int64_t rows = ceil_div(n * tp2, kOzTileA) * kOzTileA;
    const int64_t count = 2 * n * b, count_pad = ceil_div(count, kOzTileA) * kOzTileA;
    const double norm = 1.0 / ((double)n * (double)b);
    const double* x = static_cast<const double*>(x_dev);
    const double* xc = static_cast<const double*>(xc_dev);
    // aux layout: colsq[b] colxc[b] | rg[2T] | gpart[148*4*128*3] | lpart[148*4*4*16] | ecol[b]
    const size_t n_dbl = 2 * (size_t)b + 2 * (size_t)T + (size_t)FGFRFT_SMS * 4 * 128 * 3 +
                         (size_t)FGFRFT_SMS * 4 * 4 * 16;
    FGB_CUDA(c->zaux.ensure(n_dbl * sizeof(double) + (size_t)b * sizeof(int)));
    double* colsq = c->zaux.as<double>();
    double* colxc = colsq + b;
    double* rg = colxc + b;
    double* gpart = rg + 2 * T;
    double* lpart = gpart + (size_t)FGFRFT_SMS * 4 * 128 * 3;
    int* ecol = reinterpret_cast<int*>(lpart + (size_t)FGFRFT_SMS * 4 * 4 * 16);
    const int SZ = oz_zdigits();  // Z digits (bounded by column norms: one digit more than the cache)
    FGB_CUDA(c->zd.ensure((size_t)SZ * count_pad * tp2));
    // B operand of the Z GEMM (X digits) -- before waiting for Xc
    int64_t bp = 0;
    if (int st = slice_signal_rows(c, x_dev, b, &bp)) return st;
    if (int st = wait_xc(c)) return st;
    {
        ProfScope ps(KC_ELEMWISE, c->stream);
        FGB_LAUNCH(launch_colstats(x, xc, (int)n, (int)b, colsq, colxc, ecol, rg, l, c->stream), 2);
    }
    {
        OzOut o;
        o.nv = (int)(2 * b);
        o.x = x;
        o.xc = xc;
        o.l = l;
        o.epos = ecol;
        o.zd = c->zd.as<int8_t>();
        o.part = gpart;
        o.n = (int)n;
        o.tp2 = (int)tp2;
        o.kbz = (int)(tp2 / oz_bk(SZ));
        ProfScope ps(KC_I8GEMM, c->stream);
        FGB_CUDA(cudaMemsetAsync(gpart, 0, (size_t)FGFRFT_SMS * 4 * 128 * 3 * sizeof(double), c->stream));
        FGB_LAUNCH(launch_ozgemm_ex(S, 2, c->ps3.as<int8_t>(), c->pe3.as<int>(), (int)rows, c->xsl.as<int8_t>(),
                                    c->xex.as<int>(), (int)bp, (int)kp, o, c->stream),
                   1);
    }
    {
        ProfScope ps(KC_COMBINE, c->stream);
        FGB_LAUNCH(launch_gram_terms(gpart, FGFRFT_SMS, (int)tp2, l, rg, c->stream), 1);
    }
    FGB_CUDA(c->cdig.ensure((size_t)SZ * 64 * tp2));
    FGB_CUDA(c->cex.ensure(64 * (sizeof(int) + sizeof(unsigned long long))));
    const size_t width = (size_t)T;
    for (int a0 = 0; a0 < n_alpha; a0 += 64) {
        const int na = std::min(64, n_alpha - a0);
        const double* cf = coef + (size_t)a0 * width;
        int* ce = c->cex.as<int>();
        {
            OzView v{cf, (int64_t)T, 1, 0, 0, 0, na, 64, 1, (int)tp2, (int)tp2, false};
            v.tiled = 4;
            v.l = l;
            ProfScope ps(KC_SLICE, c->stream);
            FGB_LAUNCH(launch_oz_slice(v, SZ, kOzTileB, c->cdig.as<int8_t>(), ce,
                                       reinterpret_cast<unsigned long long*>(ce + 64), c->stream),
                       3);
        }
        OzOut o;
        o.c = y_dev ? static_cast<double*>(y_dev) + (size_t)a0 * count : nullptr;
        o.nv = na;
        o.x = x;
        o.xc = xc;
        o.part = lpart;
        o.c0 = cf + l;
        o.c0s = T;
        o.count = count;
        o.n = (int)n;
        o.epos = ecol;
        ProfScope ps(KC_COMBINE, c->stream);
        FGB_CUDA(cudaMemsetAsync(lpart, 0, (size_t)FGFRFT_SMS * 4 * 4 * 16 * sizeof(double), c->stream));
        FGB_LAUNCH(launch_ozgemm_ex(SZ, 3, c->zd.as<int8_t>(), nullptr, (int)count_pad, c->cdig.as<int8_t>(), ce, 64,
                                    (int)tp2, o, c->stream),
                   1);
        FGB_LAUNCH(launch_loss3(lpart, FGFRFT_SMS, na, norm, loss_dev + a0, c->stream), 1);
        FGB_LAUNCH(launch_gram_s_dlda(cf, dcoef + (size_t)a0 * width, rg, na, l, norm, s_dev + (size_t)a0 * width,
                                      dlda_dev + a0, c->stream),
                   1);
    }
    return FGFRFT_OK;
}

// MSE step over the power products: loss, s (2L+1 per order) and optionally Y.
int mse_power_route(fgfrft_cache* c, const double* coef, int n_alpha, const void* x_dev, const void* xc_dev,
                    int64_t b, void* y_dev, double* loss_dev, double* s_dev) {
    if (int st = power_products(c, x_dev, b)) return st;
    const int l = c->l;
    const size_t width = (size_t)(2 * l + 1);
    const int64_t count = 2 * c->n * b;
    const double norm = 1.0 / ((double)c->n * (double)b);
    FGB_CUDA(c->partial.ensure(combine_partial_elems(combine_max_terms()) * sizeof(double)));
    if (int st = wait_xc(c)) return st;
    for (int a0 = 0; a0 < n_alpha; a0 += 64) {
        const int na = std::min(64, n_alpha - a0);
        ProfScope ps(KC_COMBINE, c->stream);
        FGB_LAUNCH(launch_combine(gram_route(c) ? 3 : 0, c->z.as<double>(), static_cast<const double*>(x_dev),
                                  static_cast<const double*>(xc_dev), count, l, coef + (size_t)a0 * width, na, norm,
                                  y_dev ? static_cast<double*>(y_dev) + (size_t)a0 * count : nullptr,
                                  c->partial.as<double>(), s_dev + (size_t)a0 * width, loss_dev + a0, c->stream),
                   2);
    }
    return FGFRFT_OK;
}

// INT8 engine for the synthesis route's GEMMs: forced, or (auto) when the products are large
// enough to amortise the per-call digit slicing of Q / G and X.
bool use_int8_gemm(const fgfrft_cache* c, int64_t b) {
    if (!c->real || c->dtype != FGFRFT_C128 || c->n > 16384 || c->graphs > 0) return false;
    const int eng = engine_of(c);
    if (eng == FGFRFT_ENGINE_DMMA) return false;
    if (eng != FGFRFT_ENGINE_AUTO) return true;
    return c->n >= 512 && 2 * b >= 64;
}

// Small signal batches on a real cache: the fused synthesis + product kernel (Q never in HBM).
bool use_fused_apply(const fgfrft_cache* c, int n_alpha, int64_t b) {
    return c->real && c->dtype == FGFRFT_C128 && 2 * b <= rapply_fused_max_cols() && c->n <= 2048 &&
           n_alpha <= 4 && engine_of(c) == FGFRFT_ENGINE_AUTO && !c->shard && c->graphs == 0;
}

// Slice the signal block X (n x b complex) as the B operand: rows 2j + comp, K = signal index.
int slice_signal_rows(fgfrft_cache* c, const void* x_dev, int64_t b, int64_t* bp_out, cudaStream_t st) {
    if (!st) st = c->stream;
    const int S = oz_slices_default();
    const int64_t n = c->n, kp = pad_k(n), bp = ceil_div(2 * b, kOzTileB) * kOzTileB;
    FGB_CUDA(c->xsl.ensure((size_t)S * bp * kp));
    FGB_CUDA(c->xex.ensure((size_t)bp * (sizeof(int) + sizeof(unsigned long long))));
    int* xe = c->xex.as<int>();
    const OzView v{static_cast<const double*>(x_dev), 2 * n, 2, 0, 1, 0, (int)(2 * b), (int)bp, 1, (int)n, (int)kp,
                   false};
    ProfScope ps(KC_SLICE, st);
    FGB_LAUNCH(launch_oz_slice(v, S, kOzTileB, c->xsl.as<int8_t>(), xe,
                               reinterpret_cast<unsigned long long*>(xe + bp), st),
               3);
    *bp_out = bp;
    return FGFRFT_OK;
}

// Y_a = op(Q_a) X for na real m x n matrices Q_a (column-major, leading dimension ldq, stride sq
// doubles), complex X (n x b); Y_a complex m x b (leading dimension ldy, stride sy doubles).
int int8_qx_gen(fgfrft_cache* c, int na, bool inverse, const void* q, int64_t m, int64_t ldq, int64_t sq,
                const void* x_dev, int64_t b, void* y, int64_t ldy, int64_t sy, double* const* peers, int npeers,
                bool rowmax_ready, cudaEvent_t x_sliced, int64_t x_bp) {
    const int S = oz_slices_default();
    const int64_t n = c->n, mp = pad_rows(m), kp = pad_k(n), rows = (int64_t)na * mp;
    FGB_CUDA(c->qsl.ensure((size_t)S * rows * kp));
    FGB_CUDA(c->qex.ensure((size_t)rows * (sizeof(int) + sizeof(unsigned long long))));
    int* qe = c->qex.as<int>();
    {
        const double* src = static_cast<const double*>(q);
        const OzView v = inverse ? OzView{src, ldq, 1, sq, 0, 0, (int)m, (int)mp, na, (int)n, (int)kp, false}
                                 : OzView{src, 1, ldq, sq, 0, 0, (int)m, (int)mp, na, (int)n, (int)kp, true};
        ProfScope ps(KC_SLICE, c->stream);
        if (rowmax_ready)  // the producer of q left the row maxima in the rowmax half of qex
            FGB_LAUNCH(launch_oz_slice_ready(v, S, kOzTileA, c->qsl.as<int8_t>(), qe,
                                             reinterpret_cast<const unsigned long long*>(qe + rows), c->stream),
                       1);
        else
            FGB_LAUNCH(launch_oz_slice(v, S, kOzTileA, c->qsl.as<int8_t>(), qe,
                                       reinterpret_cast<unsigned long long*>(qe + rows), c->stream),
                       3);
    }
    int64_t bp = x_bp;
    if (x_sliced) {  // the caller sliced X on a side stream (node route: beside the node-operator GEMM)
        FGB_CUDA(cudaStreamWaitEvent(c->stream, x_sliced, 0));
    } else if (int st = slice_signal_rows(c, x_dev, b, &bp)) {
        return st;
    }
    ProfScope ps(KC_I8GEMM, c->stream);
    FGB_LAUNCH(launch_ozgemm(S, 1, c->qsl.as<int8_t>(), qe, (int)rows, c->xsl.as<int8_t>(), c->xex.as<int>(), (int)bp,
                             (int)kp, static_cast<double*>(y), ldy, sy, (int)m, (int)mp, (int)(2 * b), c->stream, peers,
                             npeers),
               1);
    return FGFRFT_OK;
}

int int8_qx(fgfrft_cache* c, int na, bool inverse, const void* q, const void* x_dev, int64_t b, void* y,
            bool rowmax_ready, cudaEvent_t x_sliced, int64_t x_bp) {
    return int8_qx_gen(c, na, inverse, q, c->n, c->n, c->n * c->n, x_dev, b, y, c->n, 2 * c->n * b, nullptr, 0,
                       rowmax_ready, x_sliced, x_bp);
}

// M_a = Re(G_a X^H) (real m x n, column-major ld m, stride sm) for na blocks G_a (m x b complex,
// ld m, stride 2 m b doubles), X n x b.
int int8_gx_gen(fgfrft_cache* c, int na, const void* g, int64_t m, const void* x_dev, int64_t b, void* out,
                int64_t sm) {
    const int S = oz_slices_default();
    const int64_t n = c->n, mp = pad_rows(m), kp = pad_k(2 * b), rows = (int64_t)na * mp;
    const int64_t xp = ceil_div(n, kOzTileB) * kOzTileB;
    FGB_CUDA(c->qsl.ensure((size_t)S * rows * kp));
    FGB_CUDA(c->qex.ensure((size_t)rows * (sizeof(int) + sizeof(unsigned long long))));
    FGB_CUDA(c->xsl.ensure((size_t)S * xp * kp));
    FGB_CUDA(c->xex.ensure((size_t)xp * (sizeof(int) + sizeof(unsigned long long))));
    int* ge = c->qex.as<int>();
    int* xe = c->xex.as<int>();
    {
        // G_a(i, 2j + comp) and X(l, 2j + comp): K = the (re, im) columns of the signal block
        const OzView vg{static_cast<const double*>(g), 2, 2 * m, 2 * m * b, 0, 1, (int)m, (int)mp, na, (int)(2 * b),
                        (int)kp, true};
        const OzView vx{static_cast<const double*>(x_dev), 2, 2 * n, 0, 0, 1, (int)n, (int)xp, 1, (int)(2 * b),
                        (int)kp, true};
        ProfScope ps(KC_SLICE, c->stream);
        FGB_LAUNCH(launch_oz_slice(vg, S, kOzTileA, c->qsl.as<int8_t>(), ge,
                                   reinterpret_cast<unsigned long long*>(ge + rows), c->stream),
                   3);
        FGB_LAUNCH(launch_oz_slice(vx, S, kOzTileB, c->xsl.as<int8_t>(), xe,
                                   reinterpret_cast<unsigned long long*>(xe + xp), c->stream),
                   3);
    }
    ProfScope ps(KC_I8GEMM, c->stream);
    FGB_LAUNCH(launch_ozgemm(S, 0, c->qsl.as<int8_t>(), ge, (int)rows, c->xsl.as<int8_t>(), xe, (int)xp, (int)kp,
                             static_cast<double*>(out), m, sm, (int)m, (int)mp, (int)n, c->stream),
               1);
    return FGFRFT_OK;
}

int int8_gx(fgfrft_cache* c, int na, const void* g, const void* x_dev, int64_t b, void* m) {
    return int8_gx_gen(c, na, g, c->n, x_dev, b, m, c->n * c->n);
}

// Y_a = F^(alpha_a) X over the power products (coef: the orders' c tables, inverse already folded
// in by the caller as alpha -> -alpha).
int apply_power_route(fgfrft_cache* c, const double* coef, int n_alpha, const void* x_dev, int64_t b, void* y_dev) {
    if (int st = power_products(c, x_dev, b)) return st;
    const size_t width = (size_t)(2 * c->l + 1);
    const int64_t count = 2 * c->n * b;
    for (int a0 = 0; a0 < n_alpha; a0 += 64) {
        const int na = std::min(64, n_alpha - a0);
        ProfScope ps(KC_COMBINE, c->stream);
        FGB_LAUNCH(launch_combine(1, c->z.as<double>(), static_cast<const double*>(x_dev), nullptr, count, c->l,
                                  coef + (size_t)a0 * width, na, 0.0, static_cast<double*>(y_dev) + (size_t)a0 * count,
                                  nullptr, nullptr, nullptr, c->stream),
                   1);
    }
    return FGFRFT_OK;
}

// s_aq = Re<G_a, F^(q-L) X> for all orders over the power products.
int dots_power_route(fgfrft_cache* c, int n_alpha, const void* g_dev, const void* x_dev, int64_t b, double* s_dev) {
    if (int st = power_products(c, x_dev, b)) return st;
    const size_t width = (size_t)(2 * c->l + 1);
    const int64_t count = 2 * c->n * b;
    FGB_CUDA(c->partial.ensure(combine_partial_elems(combine_max_terms()) * sizeof(double)));
    for (int a0 = 0; a0 < n_alpha; a0 += 64) {
        const int na = std::min(64, n_alpha - a0);
        ProfScope ps(KC_COMBINE, c->stream);
        FGB_LAUNCH(launch_combine(2, c->z.as<double>(), static_cast<const double*>(x_dev),
                                  static_cast<const double*>(g_dev) + (size_t)a0 * count, count, c->l, nullptr, na, 0.0,
                                  nullptr, c->partial.as<double>(), s_dev + (size_t)a0 * width, nullptr, c->stream),
                   2);
    }
    return FGFRFT_OK;
}

// c->m[a] = M_a = G_a X^H (n x n, K = b) for na orders; real cache: only M_re = Re(G X^H).
int gx_device(fgfrft_cache* c, int na, const void* g_dev, const void* x_dev, int64_t b) {
    const int n = (int)c->n;
    const size_t sl = c->mat_elems();
    if (use_int8_gemm(c, b)) return int8_gx(c, na, g_dev, x_dev, b, c->m.p);
    ProfScope ps(KC_GEMM, c->stream);
    if (c->real)
        FGB_LAUNCH(launch_rgemm(2, 2, 0, n, n, 2 * (int)b, g_dev, n, (int64_t)2 * n * b, x_dev, n, 0, c->m.p, n,
                                (int64_t)sl, na, c->stream),
                   1);
    else
        FGB_LAUNCH(gemm(c, n, n, (int)b, g_dev, n, (int64_t)n * b, false, x_dev, n, 0, true, c->m.p, n, (int64_t)sl,
                        na),
                   1);
    return FGFRFT_OK;
}

// s_dev[a][2l+1] = Re<G_a, F^k X> for all orders; g_dev n_alpha blocks of n x b.
// Order sweeps (>= 8 orders) use the DMMA split-K contraction (every byte of M and of the cache
// read once per 64 orders); a few orders use the scalar tile-pair kernel (HBM-bound).
int dots_device(fgfrft_cache* c, int n_alpha, const void* g_dev, const void* x_dev, int64_t b, double* s_dev) {
    if (use_power_route(c, n_alpha)) return dots_power_route(c, n_alpha, g_dev, x_dev, b, s_dev);
    const int n = (int)c->n;
    const size_t sl = c->mat_elems();
    const bool mma = n_alpha >= 8 && c->dtype == FGFRFT_C128;  // real caches: rdots_mma (same cap)
    const int chunk = mma ? std::min(alpha_chunk(c, n_alpha), dots_mma_max_orders()) : alpha_chunk(c, n_alpha);
    FGB_CUDA(c->m.ensure((size_t)chunk * sl * c->elem));
    FGB_CUDA(c->partial.ensure(std::max(mma ? std::max(dots_mma_partial_elems(n), rdots_mma_partial_elems(n)) : 0,
                                        dots_partial_elems(n, c->l, chunk)) *
                               sizeof(double)));
    const size_t width = (size_t)(2 * c->l + 1);
    for (int a0 = 0; a0 < n_alpha; a0 += chunk) {
        const int na = std::min(chunk, n_alpha - a0);
        if (int st = gx_device(c, na, static_cast<const char*>(g_dev) + (size_t)a0 * n * b * c->sig, x_dev, b))
            return st;
        ProfScope ps(KC_DOTS, c->stream);
        if (c->real) {
            if (na >= 8) {
                int nl = 0;
                FGB_CUDA(launch_rdots_mma(c->slabs, n, c->l, c->m.p, (int64_t)sl, na, c->partial.as<double>(),
                                          s_dev + a0 * width, c->stream, &nl));
                g_launches += nl;
            } else {
                FGB_LAUNCH(launch_rdots(c->slabs, n, c->l, c->m.p, (int64_t)sl, na, c->partial.as<double>(),
                                        s_dev + a0 * width, c->stream),
                           2);
            }
        } else if (mma && na >= 8) {
            int nl = 0;
            FGB_CUDA(launch_power_dots_mma(c->slabs, n, c->l, c->m.p, (int64_t)sl, na, c->partial.as<double>(),
                                           s_dev + a0 * width, c->stream, &nl));
            g_launches += nl;
        } else {
            FGB_LAUNCH(launch_power_dots(c->slabs, n, c->l, c->m.p, (int64_t)sl, na, c->partial.as<double>(),
                                         s_dev + a0 * width, c->stream, (int)c->elem),
                       2);
        }
    }
    return FGFRFT_OK;
}

// ------------------------------------------------------------------ memory budget of aux structures

// The reference's budget counts L n^2 16 bytes (transform.hpp:46-53); auxiliary representations
// are admitted while that count plus every admitted auxiliary byte stays within the handle's budget.
bool aux_fits(const fgfrft_cache* c, uint64_t bytes) {
    const unsigned __int128 ref = (unsigned __int128)c->l * (uint64_t)c->n * (uint64_t)c->n * 16;
    return ref + c->aux_bytes + bytes <= (unsigned __int128)c->budget;
}

// ------------------------------------------------------------------ packed step route (packed.cu)
//
// One or a few orders over a real cache with a large signal batch (config 3 / 4): Q(a) and
// dQ/da from ONE pass over the packed slabs (6 B per element instead of 8), the row maxima of
// Q / dQ left by the same kernel, one slicing pass, and ONE Ozaki GEMM [Y; dY] = [Q; dQ] X;
// loss and dL/da = 2/(NB) Re<Y - Xc, dY> from a single elementwise pass (no G, no G X^H GEMM).
bool packed_enabled(const fgfrft_cache* c) {
    static const bool off = [] {
        const char* e = std::getenv("FGFRFT_PACKED");
        return e && !std::strcmp(e, "0");
    }();
    return !off && c->real && c->dtype == FGFRFT_C128 && !c->shard && c->graphs == 0 && c->n >= 512 &&
           engine_of(c) == FGFRFT_ENGINE_AUTO;
}

// ---- the order window: node operators for the orders a caller declares it will use
//
// Q(a) is analytic in a, and over a bounded window [lo, hi] the r-point Chebyshev interpolant of its
// series coefficients matches them to 4e-15 of the largest (2e-12 for the derivatives) with r ~ 9 + 5
// (hi - lo) -- the node route's criterion (node_plan_r), here checked on 513 orders of the window.
// So Q(a) = sum_j l_j(a) W_j and dQ/da = sum_j l_j'(a) W_j with W_j = Q(x_j), exact FP64: r slabs
// instead of L powers per step (config 3, [0, 2]: 19 x 134 MB = 2.5 GB against 5.4 GB packed).
// The c_0 I terms stay out of W'_j = W_j - c_0(x_j) I: the product GEMM's epilogue adds the exact
// c_0(a), c'_0(a) (the nodiag form of the packed route).

// barycentric weights l_j(x) (and l_j'(x)) on the nodes xn with weights bw
static void bary_weights(const std::vector<double>& xn, const std::vector<double>& bw, double x, double* lj,
                         double* dj) {
    const int r = (int)xn.size();
    int hit = -1;
    for (int j = 0; j < r; ++j)
        if (std::fabs(x - xn[j]) < 1e-14 * std::max(1.0, std::fabs(x))) hit = j;
    if (hit >= 0) {  // on a node: Kronecker weights, the derivative row of the differentiation matrix
        for (int j = 0; j < r; ++j) lj[j] = j == hit ? 1.0 : 0.0;
        if (dj) {
            double diag = 0.0;
            for (int j = 0; j < r; ++j)
                if (j != hit) {
                    dj[j] = (bw[j] / bw[hit]) / (xn[hit] - xn[j]);
                    diag -= dj[j];
                }
            dj[hit] = diag;
        }
        return;
    }
    double sw = 0.0, sw2 = 0.0;
    for (int j = 0; j < r; ++j) {
        const double t = bw[j] / (x - xn[j]);
        sw += t;
        sw2 += t / (x - xn[j]);
    }
    for (int j = 0; j < r; ++j) {
        const double t = bw[j] / (x - xn[j]);
        lj[j] = t / sw;
        if (dj) dj[j] = lj[j] * (-1.0 / (x - xn[j]) + sw2 / sw);
    }
}

bool window_weights(const fgfrft_cache* c, const double* alphas, int n_alpha, bool with_d, int l_used,
                    WindowWeights* ww) {
    if (!c->win_r || l_used != c->l) return false;
    const int rows = with_d ? 2 * n_alpha : n_alpha;
    if (rows > 4) return false;
    const double eps = 1e-12 * (1.0 + std::max(std::fabs(c->win_lo), std::fabs(c->win_hi)));
    for (int a = 0; a < n_alpha; ++a)
        if (!(alphas[a] >= c->win_lo - eps && alphas[a] <= c->win_hi + eps)) return false;
    for (int a = 0; a < n_alpha; ++a)
        bary_weights(c->win_xn, c->win_bw, alphas[a], ww->w[a], with_d ? ww->w[n_alpha + a] : nullptr);
    return true;
}

// true when the packed slabs are resident (built on first use, counted against the budget).
bool ensure_packed(fgfrft_cache* c) {
    if (c->pk_state) return c->pk_state > 0;
    const uint64_t bytes = (uint64_t)packed_bytes((int)c->n, c->l);
    const uint64_t sbytes = (uint64_t)packed_scale_elems((int)c->n, c->l) * sizeof(double);
    if (!aux_fits(c, bytes + sbytes) || c->pk.ensure(bytes) != cudaSuccess || c->pks.ensure(sbytes) != cudaSuccess) {
        cudaGetLastError();
        c->pk.release();
        c->pks.release();
        c->pk_state = -1;
        return false;
    }
    // the powers' row / column maxima (the digit-emitting synthesis' row bounds): 2 L N doubles, best effort
    const uint64_t mbytes = (uint64_t)c->l * 2 * ceil_div(c->n, kTile) * kTile * sizeof(double);
    if (!aux_fits(c, bytes + sbytes + mbytes) || c->pkm.ensure(mbytes) != cudaSuccess) {
        cudaGetLastError();
        c->pkm.release();
    }
    ProfScope ps(KC_SLICE, c->stream);
    if (launch_pack_tiles(c->slabs, (int)c->n, c->l, c->pk.p, c->pks.as<double>(), c->stream,
                          c->pkm.p ? c->pkm.as<unsigned long long>() : nullptr) != cudaSuccess) {
        cudaGetLastError();
        c->pk.release();
        c->pks.release();
        c->pkm.release();
        c->pk_state = -1;
        return false;
    }
    g_launches += 1;
    c->aux_bytes += bytes + sbytes + (c->pkm.p ? mbytes : 0);
    c->pk_state = 1;
    return true;
}

// The digit cache of the tensor-core synthesis (dsynth_kernel: the same 5 B per element and power as
// the packed slabs at L = 64, a fifth of the SM issue per element, built so the synthesis could share
// the SMs with the product GEMM). Measured at config 3 it is not faster on its own (0.94 vs 0.92 ms
// synthesis, 1.70 vs 1.67 ms step) and the shell pipeline that would overlap it with the GEMM lost to
// the serial order (1.74-1.82 ms), so the packed FP64-decode synthesis (psynth) is the default and
// FGFRFT_DSYNTH=1 opts in (read per call: the tests run both engines).
static bool dsynth_wanted() {
    const char* e = std::getenv("FGFRFT_DSYNTH");
    return e && !std::strcmp(e, "1");
}

bool ensure_dsynth(fgfrft_cache* c) {
    if (!dsynth_wanted()) return false;
    if (c->ds_state) return c->ds_state > 0;
    const int64_t rows = (int64_t)dsynth_cache_rows((int)c->n), kp = dsynth_kp(c->l);
    const uint64_t bytes = (uint64_t)rows * kp * dsynth_slices(), ebytes = (uint64_t)rows * sizeof(int);
    DevBuf tmp;
    auto fail = [&] {
        cudaGetLastError();
        c->ds.release();
        c->dse.release();
        tmp.release();
        c->ds_state = -1;
        return false;
    };
    if (kp > 512 || !aux_fits(c, bytes + ebytes) || c->ds.ensure(bytes) != cudaSuccess ||
        c->dse.ensure(ebytes) != cudaSuccess || tmp.ensure((size_t)rows * sizeof(unsigned long long)) != cudaSuccess ||
        c->dsb.ensure(dsynth_coef_bytes((int)kp)) != cudaSuccess)
        return fail();
    {
        ProfScope ps(KC_SLICE, c->stream);
        if (launch_dsynth_build(static_cast<const double*>(c->slabs), (int)c->n, c->l, (int)kp, c->ds.as<int8_t>(), c->dse.as<int>(),
                                tmp.as<unsigned long long>(), c->stream) != cudaSuccess)
            return fail();
    }
    g_launches += 3;
    cudaStreamSynchronize(c->stream);  // the row-max scratch is freed below
    tmp.release();
    c->aux_bytes += bytes + ebytes;
    c->ds_state = 1;
    return true;
}

// Digits per operand of the step route's product GEMM [Y; dY] = [Q; dQ] X: 6 base-254 digits (21
// digit products). The synthesis leaves out the c_0 I term (nodiag; the GEMM epilogue adds c_0 X), so
// Q's row maxima are its off-diagonal entries rather than the diagonal c_0 ~ 0.8 (13x larger at
// config 3). Measured relative error of Y at 5 digits (15 products, 25% faster): config 3 1.9e-10
// -> 1.2e-11 with nodiag, but config 4 (N = 8192 k-NN point cloud) still 1.0e-10 -- at the 1e-10
// bar of the north star, so 5 digits is opt-in only (FGFRFT_STEP_SLICES=5); 6 digits leave ~250x.
static int step_slices() {
    static const int s = [] {
        const char* e = std::getenv("FGFRFT_STEP_SLICES");
        const int v = e ? std::atoi(e) : 6;
        return v == 5 ? 5 : 6;
    }();
    return s;
}

// The step route's cache: the digit cache when wanted and it fits, else the packed slabs.
bool ensure_step_cache(fgfrft_cache* c) { return ensure_dsynth(c) || ensure_packed(c); }

// ---- the pipelined form: row-complete shells
//
// The step is the sum of an HBM-bound pass (synthesis from the packed slabs) and a tensor-bound
// pass (the Ozaki GEMM). They overlap by ROW SHELLS: the tile pairs are enumerated I-major
// (pairs_before), so the pairs whose smaller tile index falls in a row range are one index range,
// and once it is synthesised those rows of Q (and dQ) are complete -- their row maxima, slicing and
// product rows Y[r0:r1] = Q[r0:r1, :] X can go. The synthesis + slicing of shell s+1 (side stream
// S) runs while the GEMM of shell s (stream G, high priority, persistent grid capped so the
// synthesis keeps SMs) runs; no kernel waits on another (stream events only). Shell bounds come
// from a small DP over a cost model (the first shells have the most pairs per row).
static double pk_env(const char* name, double dflt) {
    const char* e = std::getenv(name);
    return e ? std::atof(e) : dflt;
}

// Shell plan for n rows, `rows` operator blocks (1, 2, 4), b signals, L powers: DP over 128-row
// block boundaries minimising S_0 + sum_s max(sigma S_s, gamma G_(s-1)) + G_last (+ a per-shell
// launch overhead), S = synthesis + slicing of a shell, G = its GEMM. Memoised per shape.
static std::vector<PkShell> pk_plan(int64_t n, int rows, int64_t b, int l) {
    const int nt = (int)ceil_div(n, kTile);
    const int T = (int)ceil_div(n, kOzTileA);
    // Default: one shell (no overlap). Measured on B200 at config 3: the packed synthesis is
    // issue-bound per SM (FP64 decode + accumulate, ~100 SM-ms) and the GEMM tensor-bound (~115
    // SM-ms), so sharing the SMs cannot beat running them back to back by more than ~14%, and the
    // measured 4-8 shell pipelines lost 0.2-0.5 ms to the split. FGFRFT_PIPE_SHELLS
    // enables the pipeline for experiments.
    const int maxc = (int)pk_env("FGFRFT_PIPE_SHELLS", 1);
    const double hbm = 6.3e12, i8 = 3.7e15, slice_bw = 4.0e12;
    const double sigma = pk_env("FGFRFT_PIPE_SIGMA", 1.25), gamma = pk_env("FGFRFT_PIPE_GAMMA", 1.45);
    const double over = pk_env("FGFRFT_PIPE_OVERHEAD_US", 6.0) * 1e-6;
    auto tile_of = [&](int blk) { return std::min(nt, blk * (kOzTileA / kTile)); };
    auto S = [&](int a, int z) {  // synthesis + slicing of block rows [a, z)
        const double pairs = (double)(packed_pairs_before(tile_of(z), nt) - packed_pairs_before(tile_of(a), nt));
        const double rws = (double)std::min<int64_t>(n, (int64_t)z * kOzTileA) - (double)a * kOzTileA;
        return pairs * 2.0 * kTileElems * 5.0 * l / hbm + rows * rws * n * 14.0 / slice_bw;
    };
    auto G = [&](int a, int z) {
        const double rws = (double)std::min<int64_t>(n, (int64_t)z * kOzTileA) - (double)a * kOzTileA;
        return rows * rws * 2.0 * b * n * 2.0 * 21.0 / i8;
    };
    std::vector<PkShell> out;
    std::vector<int> bounds{0, T};
    if (const char* sp = std::getenv("FGFRFT_PIPE_SPLIT")) {  // explicit row fractions "f1,f2,..."
        bounds.assign(1, 0);
        for (const char* q = sp; *q;) {
            const double f = std::atof(q);
            const int blk = (int)std::lround(f * T);
            if (blk > bounds.back() && blk < T) bounds.push_back(blk);
            while (*q && *q != ',') ++q;
            if (*q == ',') ++q;
        }
        bounds.push_back(T);
    } else if (maxc > 1 && T >= 4) {
        // f[c][j][k]: best cost of shells covering blocks [0, k) with c shells, the last being [j, k)
        const double inf = 1e30;
        std::vector<double> f((size_t)(maxc + 1) * (T + 1) * (T + 1), inf);
        std::vector<int> arg(f.size(), -1);
        auto at = [&](int c, int j, int k) -> size_t { return ((size_t)c * (T + 1) + j) * (T + 1) + k; };
        for (int k = 1; k <= T; ++k) f[at(1, 0, k)] = S(0, k) + over;
        for (int c = 2; c <= maxc; ++c)
            for (int j = 1; j < T; ++j)
                for (int k = j + 1; k <= T; ++k)
                    for (int i = 0; i < j; ++i) {
                        const double pv = f[at(c - 1, i, j)];
                        if (pv >= inf) continue;
                        const double v = pv + std::max(sigma * S(j, k), gamma * G(i, j)) + over;
                        if (v < f[at(c, j, k)]) {
                            f[at(c, j, k)] = v;
                            arg[at(c, j, k)] = i;
                        }
                    }
        double best = inf;
        int bc = 1, bj = 0;
        for (int c = 1; c <= maxc; ++c)
            for (int j = 0; j < T; ++j) {
                const double v = f[at(c, j, T)];
                if (v < inf && v + G(j, T) < best) {
                    best = v + G(j, T);
                    bc = c;
                    bj = j;
                }
            }
        bounds.assign(1, T);
        int c = bc, j = bj, k = T;
        while (c >= 1) {
            bounds.push_back(j);
            const int i = arg[at(c, j, k)];
            k = j;
            j = i;
            --c;
        }
        std::reverse(bounds.begin(), bounds.end());
    }
    for (size_t s = 0; s + 1 < bounds.size(); ++s) {
        PkShell sh;
        sh.r0 = (int)std::min<int64_t>(n, (int64_t)bounds[s] * kOzTileA);
        sh.r1 = (int)std::min<int64_t>(n, (int64_t)bounds[s + 1] * kOzTileA);
        sh.p0 = (int)packed_pairs_before(tile_of(bounds[s]), nt);
        sh.p1 = (int)packed_pairs_before(tile_of(bounds[s + 1]), nt);
        if (sh.r1 > sh.r0) out.push_back(sh);
    }
    return out;
}

int ensure_pipe_streams(fgfrft_cache* c) {
    if (c->pk_g) return FGFRFT_OK;
    int lo = 0, hi = 0;
    FGB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    FGB_CUDA(cudaStreamCreateWithPriority(&c->pk_s, cudaStreamNonBlocking, lo));
    FGB_CUDA(cudaStreamCreateWithPriority(&c->pk_g, cudaStreamNonBlocking, hi));  // GEMM CTAs placed first
    for (auto* e : {&c->pk_e0, &c->pk_eg, &c->pk_ex})
        FGB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    return FGFRFT_OK;
}

// rows (1, 2 or 4) real n x n operators M_r (table rows r of coef, width coef_ld, l_used powers)
// from the packed slabs, Y_r = M_r X into y (stride 2 n b doubles), shell-pipelined.
// x_host != nullptr: X is still on the host -- it is copied into x_dev in column chunks on the
// aux stream, and the GEMM runs per chunk as its columns land, so the host->device transfer
// overlaps the synthesis (which does not need X) and the earlier chunks' products.
int64_t fused_mse_slots_per_order(int64_t n, int64_t b) {
    return (pad_rows(n) / kOzTileA) * (ceil_div(2 * b, kOzTileB) * kOzTileB / kOzTileB) * 16;
}

// Host X of the chunked step: column chunks of >= 32 signals, FGFRFT_E2E_CHUNKS (4) of them.
static void host_x_chunks(int64_t b, int* nch, int64_t* cw) {
    *nch = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)pk_env("FGFRFT_E2E_CHUNKS", 4), ceil_div(b, 32)));
    *cw = ceil_div(ceil_div(b, *nch), 32) * 32;
}

// The chunk copies of host X into x_dev on the aux stream (after everything already on c->stream:
// the previous call's readers), one event per chunk. fgfrft_mse_step calls it BEFORE its host-side
// planning (the series coefficients are ~50 us of libm on this thread), so the link starts at once.
int enqueue_host_x(fgfrft_cache* c, const double* x_host, const void* x_dev, int64_t b) {
    const int64_t n = c->n;
    int nch = 0;
    int64_t cw = b;
    host_x_chunks(b, &nch, &cw);
    if (int st = ensure_pipe_streams(c)) return st;
    if (!c->aux_stream) FGB_CUDA(cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking));
    FGB_CUDA(cudaEventRecord(c->pk_e0, c->stream));
    FGB_CUDA(cudaStreamWaitEvent(c->aux_stream, c->pk_e0, 0));  // the previous call's readers are done
    if (c->xh_ev.size() < (size_t)nch) {
        const size_t have = c->xh_ev.size();
        c->xh_ev.resize(nch, nullptr);
        for (size_t i = have; i < (size_t)nch; ++i)
            FGB_CUDA(cudaEventCreateWithFlags(&c->xh_ev[i], cudaEventDisableTiming));
    }
    for (int ch = 0; ch < nch; ++ch) {
        const int64_t j0 = ch * cw, j1 = std::min<int64_t>(b, j0 + cw);
        if (j1 <= j0) break;
        FGB_CUDA(cudaMemcpyAsync(static_cast<double*>(const_cast<void*>(x_dev)) + j0 * 2 * n, x_host + j0 * 2 * n,
                                 (size_t)(j1 - j0) * n * 16, cudaMemcpyHostToDevice, c->aux_stream));
        FGB_CUDA(cudaEventRecord(c->xh_ev[ch], c->aux_stream));
    }
    return FGFRFT_OK;
}

int packed_products(fgfrft_cache* c, const double* coef, int coef_ld, int rows, const void* x_dev, int64_t b,
                    void* y, int l_used, const double* x_host, const WindowWeights* ww, const double* fuse_xc,
                    double* fuse_part, bool* fused) {
    if (fused) *fused = false;
    const int S = step_slices();
    const int64_t n = c->n, mp = pad_rows(n), sl = n * n, kp = pad_k(n);
    const int64_t bp = ceil_div(2 * b, kOzTileB) * kOzTileB;
    const char* split = std::getenv("FGFRFT_PIPE_SPLIT");
    const uint64_t key = ((uint64_t)n << 40) ^ ((uint64_t)rows << 32) ^ ((uint64_t)b << 8) ^ (uint64_t)l_used ^
                         ((uint64_t)pk_env("FGFRFT_PIPE_SHELLS", 1) << 56) ^ ((uint64_t)dsynth_wanted() << 62) ^
                         (split ? std::hash<std::string>{}(split) : 0);
    if (c->pk_plan_key != key) {
        c->pk_plan = pk_plan(n, rows, b, l_used);
        c->pk_plan_key = key;
    }
    if (x_host && c->pk_plan.size() > 1) {  // the chunked host-X form runs one shell
        c->pk_plan.assign(1, PkShell{0, (int)n, 0, -1});
        c->pk_plan_key = 0;
    }
    // the window synthesis has no pair coupling: row shells are plain row ranges (FGFRFT_WIN_SHELLS
    // equal shells; 1 = serial, the default: measured at config 3 on [0, 2], 2 / 3 / 4 shells with the
    // GEMM capped at 100-132 CTAs took 1.44-1.75 ms against 1.45 serial -- the GEMM loses to the
    // shared SMs what the overlap hides)
    std::vector<PkShell> wplan;
    if (ww) {
        const int T = (int)ceil_div(n, kOzTileA);
        const int k = x_host ? 1 : std::max(1, std::min(T, (int)pk_env("FGFRFT_WIN_SHELLS", 1)));
        for (int s = 0; s < k; ++s) {
            const int b0 = (int)((int64_t)T * s / k), b1 = (int)((int64_t)T * (s + 1) / k);
            wplan.push_back(PkShell{(int)std::min<int64_t>(n, (int64_t)b0 * kOzTileA),
                                    (int)std::min<int64_t>(n, (int64_t)b1 * kOzTileA), 0, 0});
        }
    }
    const std::vector<PkShell>& plan = ww ? wplan : c->pk_plan;
    int64_t srows = 0;  // sliced rows over all shells (each shell padded to 128)
    for (const PkShell& sh : plan) srows += pad_rows(sh.r1 - sh.r0);
    const int64_t exps_ints = ceil_div((int64_t)rows * srows, 2) * 2;
    FGB_CUDA(c->q.ensure((size_t)rows * sl * sizeof(double)));
    FGB_CUDA(c->qsl.ensure((size_t)S * rows * srows * kp));
    FGB_CUDA(c->qex.ensure((size_t)exps_ints * sizeof(int) + (size_t)rows * mp * sizeof(unsigned long long)));
    FGB_CUDA(c->xsl.ensure((size_t)S * bp * kp));
    FGB_CUDA(c->xex.ensure((size_t)bp * (sizeof(int) + sizeof(unsigned long long))));
    if (int st = ensure_pipe_streams(c)) return st;
    int* exps = c->qex.as<int>();
    unsigned long long* rmax = reinterpret_cast<unsigned long long*>(exps + exps_ints);
    double* q = c->q.as<double>();
    FGB_CUDA(cudaEventRecord(c->pk_e0, c->stream));
    FGB_CUDA(cudaStreamWaitEvent(c->pk_s, c->pk_e0, 0));
    FGB_CUDA(cudaStreamWaitEvent(c->pk_g, c->pk_e0, 0));
    // host X: column chunks of >= 32 signals (64 B-operand rows) copied on the aux stream
    int nch = 0;
    int64_t cw = b;
    if (x_host) {
        host_x_chunks(b, &nch, &cw);
        if (c->xh_pre == x_host) {  // fgfrft_mse_step enqueued them before its host-side planning
            c->xh_pre = nullptr;
        } else if (int st = enqueue_host_x(c, x_host, x_dev, b)) {
            return st;
        }
        c->xh_pre = nullptr;
    }
    // G: X sliced once (B operand: rows 2j + comp, K = signal index), while S synthesises shell 0
    if (!x_host) {
        int* xe = c->xex.as<int>();
        const OzView v{static_cast<const double*>(x_dev), 2 * n, 2, 0, 1, 0, (int)(2 * b), (int)bp, 1, (int)n,
                       (int)kp, false};
        ProfScope ps(KC_SLICE, c->pk_g);
        FGB_LAUNCH(launch_oz_slice(v, S, kOzTileB, c->xsl.as<int8_t>(), xe,
                                   reinterpret_cast<unsigned long long*>(xe + bp), c->pk_g),
                   3);
    }
    // synthesis engine: the window's node operators, tensor-core digits (dsynth) or the packed FP64
    // decode (psynth)
    const bool tc = !ww && dsynth_wanted() && c->ds_state > 0;
    c->pk_tc = tc;
    c->pk_win = ww != nullptr;
    if (!ww && !tc && !ensure_packed(c)) return FGFRFT_CAPACITY;
    // psynth emits [Q; dQ]'s digits itself (row exponents from the power maxima, prow_bound_kernel):
    // one order, one shell, whole 128-row tiles (FGFRFT_PSYNTH_DIGITS=0: FP64 Q + the slicing pass)
    const bool emit = !ww && !tc && plan.size() == 1 && rows == 2 && n % kOzTileA == 0 && c->pkm.p &&
                      oz_bk(S) == 64 && pk_env("FGFRFT_PSYNTH_DIGITS", 1) != 0;
    c->pk_emit = emit;
    if (!emit) FGB_CUDA(cudaMemsetAsync(rmax, 0, (size_t)rows * mp * sizeof(unsigned long long), c->pk_s));
    const int64_t dkp = dsynth_kp(c->l);
    if (tc) {
        ProfScope ps(KC_SYNTH, c->pk_s);
        FGB_LAUNCH(launch_dsynth_coefs(coef, coef_ld, l_used, rows, (int)dkp, c->dsb.as<int8_t>(), c->pk_s), 1);
    }
    const int gcap = (int)pk_env("FGFRFT_PIPE_GEMM_CTAS", 100);
    const int syn_cap = (int)pk_env("FGFRFT_PIPE_SYN_CTAS", FGFRFT_SMS - gcap);  // one CTA per SM
    if (c->pk_es.size() < plan.size()) {
        const size_t have = c->pk_es.size();
        c->pk_es.resize(plan.size(), nullptr);
        for (size_t i = have; i < plan.size(); ++i)
            FGB_CUDA(cudaEventCreateWithFlags(&c->pk_es[i], cudaEventDisableTiming));
    }
    // [Y; dY] rows of shell / chunk: the synthesis leaves out c_0 I (nodiag), the GEMM epilogue adds
    // c_0 X (Q's row maxima then follow its off-diagonal entries: at config 3, alpha = 0.37, the
    // diagonal is 0.80 against 0.06 off it, and the 5-digit slicing error drops 1.9e-10 -> 1.2e-11)
    auto gemm_out = [&](double* yp, int64_t rv, int64_t rp, int64_t nv, const double* xp, int max_ctas) {
        OzOut o;
        o.c = yp;
        o.ldc = n;
        o.sc = 2 * n * b;
        o.mv = (int)rv;
        o.mp = (int)rp;
        o.nv = (int)nv;
        o.max_ctas = max_ctas;
        o.dx = xp;
        o.dgc = coef + l_used;
        o.dgs = coef_ld;
        return o;
    };
    int64_t row_off = 0;
    for (size_t s = 0; s < plan.size(); ++s) {
        const PkShell& sh = plan[s];
        const int64_t rv = sh.r1 - sh.r0, rp = pad_rows(rv);
        int8_t* dst = c->qsl.as<int8_t>() + (size_t)S * rows * row_off * kp;
        int* ex = exps + rows * row_off;
        if (emit) {
            {
                ProfScope ps(KC_SLICE, c->pk_s);
                FGB_LAUNCH(launch_prow_bound(c->pkm.as<unsigned long long>(), (int)n, l_used, coef, coef_ld, rows,
                                             (int)rp, ex, c->pk_s),
                           1);
            }
            ProfScope ps(KC_SYNTH, c->pk_s);
            FGB_LAUNCH(launch_psynth(c->pk.p, c->pks.as<double>(), (int)n, l_used, c->l, coef, coef_ld, rows, nullptr, 0,
                                     nullptr, 0, c->pk_s, sh.p0, sh.p1, 0, 0, 1, dst, ex, (int)rp, (int)kp, S),
                       1);
        } else {
            ProfScope ps(KC_SYNTH, c->pk_s);
            // shell 0 runs alone (the GEMM has nothing yet): full grid; later shells share the GPU
            if (ww)
                FGB_LAUNCH(launch_window_synth(c->win.as<double>(), c->win_r, (int)n, *ww, rows, q, sl, rmax, mp,
                                               c->pk_s, sh.r0, sh.r1),
                           1);
            else if (tc)
                FGB_LAUNCH(launch_dsynth(c->ds.as<int8_t>(), c->dse.as<int>(), c->dsb.as<int8_t>(), (int)dkp, (int)n,
                                         sh.p0, sh.p1, coef, coef_ld, l_used, rows, q, sl, rmax, mp,
                                         s == 0 ? (int)pk_env("FGFRFT_SYN_CAP0", 0) : syn_cap, c->pk_s, 1),
                           1);
            else
                FGB_LAUNCH(launch_psynth(c->pk.p, c->pks.as<double>(), (int)n, l_used, c->l, coef, coef_ld, rows, q, sl,
                                         rmax, mp, c->pk_s, sh.p0, sh.p1, s == 0 ? 0 : syn_cap, 0, 1),
                           1);
        }
        if (!emit) {
            OzView v{q + sh.r0, 1, n, sl, 0, 0, (int)rv, (int)rp, rows, (int)n, (int)kp, true};
            v.rmb = mp;
            ProfScope ps(KC_SLICE, c->pk_s);
            FGB_LAUNCH(launch_oz_slice_ready(v, S, kOzTileA, dst, ex, rmax + sh.r0, c->pk_s), 1);
        }
        FGB_CUDA(cudaEventRecord(c->pk_es[s], c->pk_s));
        if (x_host) {  // one shell: per X chunk, slice its columns, then their products
            for (int ch = 0; ch < nch; ++ch) {
                const int64_t j0 = ch * cw, j1 = std::min<int64_t>(b, j0 + cw);
                if (j1 <= j0) break;
                const int64_t crows = 2 * (j1 - j0), cp = ceil_div(crows, kOzTileB) * kOzTileB;
                int* xe = c->xex.as<int>() + 2 * j0;
                int8_t* xd = c->xsl.as<int8_t>() + (size_t)2 * j0 * kp * S;
                FGB_CUDA(cudaStreamWaitEvent(c->pk_g, c->xh_ev[ch], 0));
                {
                    const OzView v{static_cast<const double*>(x_dev) + j0 * 2 * n, 2 * n, 2, 0, 1, 0, (int)crows,
                                   (int)cp, 1, (int)n, (int)kp, false};
                    ProfScope ps(KC_SLICE, c->pk_g);
                    FGB_LAUNCH(launch_oz_slice(v, S, kOzTileB, xd, xe, nullptr, c->pk_g), 1);
                }
                if (ch == 0) FGB_CUDA(cudaStreamWaitEvent(c->pk_g, c->pk_es[s], 0));
                ProfScope ps(KC_I8GEMM, c->pk_g);
                FGB_LAUNCH(launch_ozgemm_ex(S, 1, dst, ex, (int)(rows * rp), xd, xe, (int)cp, (int)kp,
                                            gemm_out(static_cast<double*>(y) + 2 * sh.r0 + j0 * 2 * n, rv, rp, crows,
                                                     static_cast<const double*>(x_dev) + 2 * sh.r0 + j0 * 2 * n, 0),
                                            c->pk_g),
                           1);
            }
            row_off += rp;
            continue;
        }
        FGB_CUDA(cudaStreamWaitEvent(c->pk_g, c->pk_es[s], 0));
        {
            ProfScope ps(KC_I8GEMM, c->pk_g);
            const bool last = s + 1 == plan.size();
            OzOut o = gemm_out(static_cast<double*>(y) + 2 * sh.r0, rv, rp, 2 * b,
                               static_cast<const double*>(x_dev) + 2 * sh.r0, last ? 0 : gcap);
            // fused MSE: one shell of [Q_a; dQ_a] rows (rows = 2 n_alpha blocks), the loss pass in the
            // epilogue (dY is never stored)
            if (fuse_xc && fuse_part && plan.size() == 1 && rows % 2 == 0) {
                o.lpart = fuse_part;
                o.lxc = fuse_xc + 2 * sh.r0;
                if (fused) *fused = true;
            }
            FGB_LAUNCH(launch_ozgemm_ex(S, 1, dst, ex, (int)(rows * rp), c->xsl.as<int8_t>(), c->xex.as<int>(), (int)bp,
                                        (int)kp, o, c->pk_g),
                       1);
        }
        row_off += rp;
    }
    FGB_CUDA(cudaEventRecord(c->pk_eg, c->pk_g));
    FGB_CUDA(cudaStreamWaitEvent(c->stream, c->pk_eg, 0));
    return FGFRFT_OK;
}

int mse_packed_step(fgfrft_cache* c, const double* coef, int n_alpha, const void* x_dev, const void* xc_dev, int64_t b,
                    void* y_dev, double* loss_dev, double* dlda_dev, const WindowWeights* ww, const double* x_host,
                    const double* xc_host) {
    const int64_t n = c->n, blk = 2 * n * b;  // doubles per n x b complex block
    const int rows = 2 * n_alpha;             // table rows [c(a_0) ..][c'(a_0) ..]: Q_a then dQ_a
    FGB_CUDA(c->ydy.ensure((size_t)rows * blk * sizeof(double)));
    // device-resident step: the loss pass rides in the product GEMM's epilogue (FGFRFT_FUSED_MSE=0:
    // the separate mse_dy pass). The host-X form keeps the separate pass: Xc lands last there.
    const bool want_fuse = !x_host && pk_env("FGFRFT_FUSED_MSE", 1) != 0 &&
                           (ww ? pk_env("FGFRFT_WIN_SHELLS", 1) <= 1 : pk_env("FGFRFT_PIPE_SHELLS", 1) <= 1);
    const int64_t per = fused_mse_slots_per_order(n, b);
    if (want_fuse) FGB_CUDA(c->lpart.ensure((size_t)n_alpha * per * 2 * sizeof(double)));
    bool fused = false;
    void* yd = want_fuse && y_dev ? y_dev : c->ydy.p;  // fused: Y lands in the caller's buffer directly
    if (int st = packed_products(c, coef, 2 * c->l + 1, rows, x_dev, b, yd, c->l, x_host, ww,
                                 want_fuse ? static_cast<const double*>(xc_dev) : nullptr,
                                 want_fuse ? c->lpart.as<double>() : nullptr, &fused))
        return st;
    if (fused) {
        const double norm = 1.0 / ((double)n * (double)b);
        ProfScope ps(KC_ELEMWISE, c->stream);
        FGB_LAUNCH(launch_fused_mse_finish(c->lpart.as<double>(), per, n_alpha, norm, loss_dev, dlda_dev, c->stream), 1);
        c->last_route = c->pk_win ? 5 : c->pk_tc ? 4 : 3;
        c->last_nodes = c->pk_win ? c->win_r : 0;
        return FGFRFT_OK;
    }
    if (yd != c->ydy.p) {  // not fused after all (a multi-shell plan): Y and dY in the step buffer
        if (int st = packed_products(c, coef, 2 * c->l + 1, rows, x_dev, b, c->ydy.p, c->l, x_host, ww)) return st;
    }
    const double norm = 1.0 / ((double)n * (double)b);
    if (xc_host) {
        // Xc behind X on the aux stream, in 4 column chunks like X (one 67 MB pinned copy measured 46 GB/s
        // on this pool against 55 GB/s chunked, tools/probes/h2d_probe.py); the loss pass runs per chunk
        // as it lands, so only the last chunk's quarter is left once the host link goes quiet
        constexpr int kXcChunks = 4;
        if (c->xch_ev.size() < (size_t)kXcChunks) {
            const size_t have = c->xch_ev.size();
            c->xch_ev.resize(kXcChunks, nullptr);
            for (size_t i = have; i < (size_t)kXcChunks; ++i)
                FGB_CUDA(cudaEventCreateWithFlags(&c->xch_ev[i], cudaEventDisableTiming));
        }
        const int64_t ce = ceil_div(b, (int64_t)kXcChunks) * n;  // complex elements per chunk (whole columns)
        int nq = 0;
        for (int64_t e0 = 0; e0 < n * b; e0 += ce, ++nq) {
            FGB_CUDA(cudaMemcpyAsync(static_cast<double*>(const_cast<void*>(xc_dev)) + 2 * e0, xc_host + 2 * e0,
                                     (size_t)std::min(ce, n * b - e0) * 16, cudaMemcpyHostToDevice, c->aux_stream));
            FGB_CUDA(cudaEventRecord(c->xch_ev[nq], c->aux_stream));
        }
        FGB_CUDA(c->lpart.ensure((size_t)n_alpha * nq * mse_dy_part_elems() * sizeof(double)));
        ProfScope ps(KC_ELEMWISE, c->stream);
        int q = 0;
        for (int64_t e0 = 0; e0 < n * b; e0 += ce, ++q) {
            const int64_t cnt = std::min(ce, n * b - e0);
            FGB_CUDA(cudaStreamWaitEvent(c->stream, c->xch_ev[q], 0));
            for (int a = 0; a < n_alpha; ++a) {
                const double* ya = c->ydy.as<double>() + (size_t)a * blk + 2 * e0;
                FGB_LAUNCH(launch_mse_dy_part(ya, ya + (size_t)n_alpha * blk, static_cast<const double*>(xc_dev) + 2 * e0,
                                              cnt, y_dev ? static_cast<double*>(y_dev) + (size_t)a * blk + 2 * e0 : nullptr,
                                              c->lpart.as<double>(), a * nq + q, c->stream),
                           1);
            }
        }
        for (int a = 0; a < n_alpha; ++a)
            FGB_LAUNCH(launch_mse_dy_finish_n(c->lpart.as<double>() + (size_t)a * nq * mse_dy_part_elems(), nq, norm,
                                              loss_dev + a, dlda_dev + a, c->stream),
                       1);
    } else {
        if (int st = wait_xc(c)) return st;
        FGB_CUDA(c->lpart.ensure(mse_dy_part_elems() * sizeof(double)));
        ProfScope ps(KC_ELEMWISE, c->stream);
        for (int a = 0; a < n_alpha; ++a) {
            const double* ya = c->ydy.as<double>() + (size_t)a * blk;
            FGB_LAUNCH(launch_mse_dy(ya, ya + (size_t)n_alpha * blk, xc_dev, n * b,
                                     y_dev ? static_cast<double*>(y_dev) + (size_t)a * blk : nullptr,
                                     c->lpart.as<double>(), norm, loss_dev + a, dlda_dev + a, c->stream),
                       2);
        }
    }
    c->last_route = c->pk_win ? 5 : c->pk_tc ? 4 : 3;
    c->last_nodes = c->pk_win ? c->win_r : 0;
    return FGFRFT_OK;
}

}  // namespace fgbi

// ===================================================================================== C ABI

extern "C" {

const char* fgfrft_last_error(void) { return g_err.c_str(); }

const char* fgfrft_version(void) { return "0.1.0-b200"; }

uint64_t fgfrft_launch_count(void) { return g_launches.load(); }

int fgfrft_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = on != 0;
    return FGFRFT_OK;
}

int fgfrft_profile_read(double* ms, int64_t* counts, int reset) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (int k = 0; k < KC_COUNT; ++k) {
        if (ms) ms[k] = 0.0;
        if (counts) counts[k] = 0;
    }
    for (const ProfRec& r : g_prof) {
        if (r.cls < 0 || r.cls >= KC_COUNT) continue;
        FGB_CUDA(cudaEventSynchronize(r.b));
        float t = 0.f;
        FGB_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
        if (ms) ms[r.cls] += t;
        if (counts) counts[r.cls] += 1;
    }
    if (reset) {
        for (const ProfRec& r : g_prof) {
            g_prof_pool.push_back(r.a);
            g_prof_pool.push_back(r.b);
        }
        g_prof.clear();
    }
    return FGFRFT_OK;
}

int fgfrft_profile_trace(int* cls, double* t0, double* t1, int cap, int* count) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    const int m = (int)g_prof.size();
    if (count) *count = m;
    for (int i = 0; i < m && i < cap; ++i) {
        const ProfRec& r = g_prof[i];
        FGB_CUDA(cudaEventSynchronize(r.b));
        float a = 0.f, b = 0.f;
        FGB_CUDA(cudaEventElapsedTime(&a, g_prof[0].a, r.a));
        FGB_CUDA(cudaEventElapsedTime(&b, g_prof[0].a, r.b));
        if (cls) cls[i] = r.cls;
        if (t0) t0[i] = a;
        if (t1) t1[i] = b;
    }
    return FGFRFT_OK;
}

int fgfrft_sinc_coeffs(double alpha, int l, double* c, double* dc) {
    if (l < 1) return fail(FGFRFT_PARAMETER, "sinc_coeffs: truncation order must be >= 1");
    host_sinc_coeffs(alpha, l, c, dc);
    return FGFRFT_OK;
}

uint64_t fgfrft_fnv1a64(const void* data, size_t nbytes) { return host_fnv1a64(data, nbytes); }

int fgfrft_cache_create(const double* f, int64_t n, int l, uint64_t memory_budget, int dtype, int device,
                        fgfrft_cache** out) {
    FGB_GUARD_BEGIN
    fgfrft_cache* c = nullptr;
    if (int st = create_common(f, n, l, memory_budget, dtype, device, out, &c)) return st;
    DeviceGuard dg(device);
    if (int st = build_powers(c, f)) {
        destroy_cache(c);
        return st;
    }
    *out = c;
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_cache_create_from_powers(const double* powers, const double* f, int64_t n, int l, uint64_t memory_budget,
                                    int dtype, int device, fgfrft_cache** out) {
    FGB_GUARD_BEGIN
    if (!powers) return fail(FGFRFT_PARAMETER, "null powers");
    fgfrft_cache* c = nullptr;
    if (int st = create_common(f, n, l, memory_budget, dtype, device, out, &c)) return st;
    DeviceGuard dg(device);
    if (int st = upload_powers(c, powers)) {
        destroy_cache(c);
        return st;
    }
    *out = c;
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_cache_destroy(fgfrft_cache* cache) {
    FGB_GUARD_BEGIN
    destroy_cache(cache);
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_cache_info(const fgfrft_cache* c, int64_t* n, int* l, uint64_t* fingerprint, int* dtype, int* device) {
    if (int st = check_handle(c)) return st;
    if (n) *n = c->n;
    if (l) *l = c->l;
    if (fingerprint) *fingerprint = c->fingerprint;
    if (dtype) *dtype = c->api_c64 ? FGFRFT_C64 : c->dtype;
    if (device) *device = c->device;
    return FGFRFT_OK;
}

int fgfrft_cache_route_info(const fgfrft_cache* c, int* route, int* nodes) {
    if (int st = check_handle(c)) return st;
    if (route) *route = c->last_route;
    if (nodes) *nodes = c->last_nodes;
    return FGFRFT_OK;
}

int fgfrft_cache_is_real(const fgfrft_cache* c, int* real) {
    if (int st = check_handle(c)) return st;
    if (real) *real = c->real ? 1 : 0;
    return FGFRFT_OK;
}

int fgfrft_cache_power(fgfrft_cache* c, int k, double* out) {
    FGB_GUARD_BEGIN
    if (int st = check_handle(c)) return st;
    if (k < 1 || k > c->l) return fail(FGFRFT_PARAMETER, "PowerCache: power index out of range");
    if (!out) return fail(FGFRFT_PARAMETER, "null output");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    FGB_CUDA(c->tmp.ensure(c->mat_elems() * 16));
    if (c->real)
        FGB_LAUNCH(launch_rfrom_tiled(c->slab(k), c->tmp.p, (int)c->n, c->stream), 1);
    else
        FGB_LAUNCH(launch_from_tiled(c->slab(k), c->tmp.p, (int)c->n, (int)c->elem, c->stream), 1);
    FGB_CUDA(cudaMemcpyAsync(out, c->tmp.p, c->mat_elems() * 16, cudaMemcpyDeviceToHost, c->stream));
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_cache_verify(const fgfrft_cache* c, const double* f) {
    if (int st = check_handle(c)) return st;
    if (!f) return fail(FGFRFT_PARAMETER, "null matrix");
    if (host_fnv1a64(f, c->mat_elems() * 16) != c->fingerprint)
        return fail(FGFRFT_NUMERICAL, "PowerCache: fingerprint mismatch, cache is stale for this matrix");
    return FGFRFT_OK;
}

int fgfrft_cache_set_stream(fgfrft_cache* c, void* stream) {
    if (int st = check_handle(c)) return st;
    std::lock_guard<std::mutex> lk(c->mu);
    c->stream = static_cast<cudaStream_t>(stream);  // NULL = the CUDA default stream
    return FGFRFT_OK;
}

int fgfrft_cache_set_engine(fgfrft_cache* c, int engine) {
    if (int st = check_handle(c)) return st;
    if (engine < FGFRFT_ENGINE_AUTO || engine > FGFRFT_ENGINE_INT8_COMBINE)
        return fail(FGFRFT_PARAMETER, "unknown engine");
    std::lock_guard<std::mutex> lk(c->mu);
    c->engine = engine;
    return FGFRFT_OK;
}

int fgfrft_cache_orthogonality(const fgfrft_cache* c, double* residual) {
    if (int st = check_handle(c)) return st;
    if (residual) *residual = c->ortho_residual;
    return FGFRFT_OK;
}

int fgfrft_cache_set_order_window(fgfrft_cache* c, double lo, double hi) {
    FGB_GUARD_BEGIN
    if (int st = check_handle(c)) return st;
    if (!std::isfinite(lo) || !std::isfinite(hi)) return fail(FGFRFT_PARAMETER, "order window: bounds must be finite");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    if (c->win_r) {
        c->aux_bytes -= (uint64_t)c->win_r * c->n * c->n * 8;
        c->win.release();
        c->win_r = 0;
        c->win_xn.clear();
        c->win_bw.clear();
    }
    if (!(hi > lo)) return FGFRFT_OK;  // cleared
    if (!packed_enabled(c)) return fail(FGFRFT_PARAMETER, "order window: needs the packed step route (real F, n >= 512)");
    const int l = c->l, T = 2 * l + 1, ns = 513;
    std::vector<double> al((size_t)ns), coefs((size_t)2 * ns * T);
    for (int i = 0; i < ns; ++i) {
        al[i] = lo + (hi - lo) * (double)i / (double)(ns - 1);
        host_sinc_coeffs_fast(al[i], l, &coefs[(size_t)i * T], &coefs[(size_t)(ns + i) * T]);
    }
    std::vector<double> tab, d0, pw;
    int r = 0, rp = 0;
    for (int rr = std::max(6, (int)std::floor(8.0 + 4.2 * (hi - lo))); rr <= kWindowMaxNodes; ++rr)
        if (node_plan_r(al.data(), ns, l, true, coefs.data(), rr, tab, d0, pw, &rp)) {
            r = rr;
            break;
        }
    if (!r) return fail(FGFRFT_PARAMETER, "order window: too wide for 48 interpolation nodes");
    const uint64_t bytes = (uint64_t)r * c->n * c->n * 8;
    if (!aux_fits(c, bytes)) return fail(FGFRFT_CAPACITY, "order window: node operators exceed the memory budget");
    for (int j = 0; j < r; ++j) tab[(size_t)j * T + l] = 0.0;  // W'_j: c_0 I left out
    DevBuf tmp;
    FGB_CUDA(tmp.ensure(tab.size() * 8));
    FGB_CUDA(c->win.ensure(bytes));
    FGB_CUDA(cudaMemcpyAsync(tmp.p, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, c->stream));
    if (int st = synth_into(c, tmp.as<double>(), r, l, c->win.p, true)) return st;
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    c->win_xn.resize(r);
    c->win_bw.resize(r);
    const double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
    for (int j = 0; j < r; ++j) {  // the nodes node_plan_r interpolated on
        const double th = M_PI * (2.0 * j + 1.0) / (2.0 * r);
        c->win_xn[j] = mid + half * std::cos(th);
        c->win_bw[j] = ((j & 1) ? -1.0 : 1.0) * std::sin(th);
    }
    c->win_lo = lo;
    c->win_hi = hi;
    c->win_r = r;
    c->aux_bytes += bytes;
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_cache_order_window(const fgfrft_cache* c, double* lo, double* hi, int* nodes) {
    if (!c) return fail(FGFRFT_PARAMETER, "null cache handle");
    if (lo) *lo = c->win_lo;
    if (hi) *hi = c->win_hi;
    if (nodes) *nodes = c->win_r;
    return FGFRFT_OK;
}

int fgfrft_cache_prepare(fgfrft_cache* c) {
    FGB_GUARD_BEGIN
    if (int st = check_handle(c)) return st;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    // every structure a route may build lazily, in the order the routes prefer them, each only while
    // it fits the handle's memory budget (aux_fits): the packed slabs (one / two-order steps), the
    // element-row digit slices (node-interpolated sweeps), the stacked digit slices (power route)
    if (packed_enabled(c)) ensure_step_cache(c);
    if (c->real && c->dtype == FGFRFT_C128 && engine_of(c) != FGFRFT_ENGINE_DMMA &&
        2 * c->l + 1 <= combine_max_terms()) {
        if (engine_of(c) == FGFRFT_ENGINE_AUTO && !c->es_slices && aux_fits(c, elem_slice_bytes(c)))
            if (int st = ensure_elem_slices(c)) return st;
        if (!c->ps_slices && aux_fits(c, power_slice_bytes(c)))
            if (int st = ensure_power_slices(c)) return st;
        if (use_int8_combine(c))
            if (int st = ensure_power_slices3(c)) return st;
    }
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_cache_device_slab(fgfrft_cache* c, int k, void** dptr) {
    if (int st = check_handle(c)) return st;
    if (k < 1 || k > c->l) return fail(FGFRFT_PARAMETER, "PowerCache: power index out of range");
    *dptr = c->slab(k);
    return FGFRFT_OK;
}

int fgfrft_cache_device_bytes(const fgfrft_cache* c, uint64_t* bytes) {
    if (int st = check_handle(c)) return st;
    *bytes = (uint64_t)c->slab_bytes() * (uint64_t)c->l;  // padded tiled slabs
    return FGFRFT_OK;
}

int fgfrft_synthesize_dev(fgfrft_cache* c, const double* alphas, int n_alpha, int truncation, int which,
                          void* out_dev) {
    FGB_GUARD_BEGIN
    if (int st = check_handle(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (which != FGFRFT_Q && which != FGFRFT_DQ) return fail(FGFRFT_PARAMETER, "which must be FGFRFT_Q or FGFRFT_DQ");
    int l_used = 0;
    if (int st = resolve_truncation(c, truncation, which, &l_used)) return st;
    if (!out_dev) return fail(FGFRFT_PARAMETER, "null output");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    double* coef = nullptr;
    if (int st = upload_coefs(c, alphas, n_alpha, l_used, &coef)) return st;
    const double* table = which == FGFRFT_Q ? coef : coef + (size_t)n_alpha * (2 * l_used + 1);
    if (c->api_c64 && !tl_internal_signals) {  // complex64 output
        const size_t cnt = (size_t)n_alpha * c->mat_elems();
        FGB_CUDA(c->by.ensure(cnt * 16));
        if (int st = synth_into(c, table, n_alpha, l_used, c->by.p)) return st;
        FGB_LAUNCH(launch_demote(c->by.p, out_dev, (int64_t)cnt, c->stream), 1);
        return FGFRFT_OK;
    }
    return synth_into(c, table, n_alpha, l_used, out_dev);
    FGB_GUARD_END
}

int fgfrft_synthesize(fgfrft_cache* c, const double* alphas, int n_alpha, int truncation, int which, double* out) {
    FGB_GUARD_BEGIN
    if (int st = check_handle(c)) return st;
    if (!out) return fail(FGFRFT_PARAMETER, "null output");
    if (int st = check_alphas(alphas, n_alpha)) return st;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        DeviceGuard dg(c->device);
        FGB_CUDA(c->y.ensure((size_t)n_alpha * c->mat_elems() * (c->real ? 16 : c->elem)));
    }
    {
        InternalSignals internal;
        if (int st = fgfrft_synthesize_dev(c, alphas, n_alpha, truncation, which, c->y.p)) return st;
    }
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    return download_as_c128(c, c->y.p, (size_t)n_alpha * c->mat_elems(), out);
    FGB_GUARD_END
}

int fgfrft_apply_dev(fgfrft_cache* c, const double* alphas, int n_alpha, int truncation, int inverse,
                     const void* x_dev, int64_t b, void* y_dev) {
    FGB_GUARD_BEGIN
    if (int st = check_handle(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (b < 0) return fail(FGFRFT_SHAPE, "apply_forward: negative signal count");
    int l_used = 0;
    if (int st = resolve_truncation(c, truncation, FGFRFT_Q, &l_used)) return st;
    if (b == 0) return FGFRFT_OK;
    if (!x_dev || !y_dev) return fail(FGFRFT_PARAMETER, "null signal buffer");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    if (c->api_c64 && !tl_internal_signals) {  // complex64 signals in and out
        const size_t xe = (size_t)c->n * b;
        FGB_CUDA(c->bx.ensure(xe * 16));
        FGB_CUDA(c->by.ensure(xe * n_alpha * 16));
        FGB_LAUNCH(launch_promote(x_dev, c->bx.p, (int64_t)xe, c->stream), 1);
        if (int st = apply_device(c, alphas, n_alpha, l_used, inverse != 0, c->bx.p, b, c->by.p)) return st;
        FGB_LAUNCH(launch_demote(c->by.p, y_dev, (int64_t)(xe * n_alpha), c->stream), 1);
        return FGFRFT_OK;
    }
    return apply_device(c, alphas, n_alpha, l_used, inverse != 0, x_dev, b, y_dev);
    FGB_GUARD_END
}

int fgfrft_apply(fgfrft_cache* c, const double* alphas, int n_alpha, int truncation, int inverse, const double* x,
                 int64_t b, double* y) {
    FGB_GUARD_BEGIN
    if (int st = check_handle(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (b < 0) return fail(FGFRFT_SHAPE, "apply_forward: negative signal count");
    int l_used = 0;
    if (int st = resolve_truncation(c, truncation, FGFRFT_Q, &l_used)) return st;
    if (b == 0) return FGFRFT_OK;
    if (!x || !y) return fail(FGFRFT_PARAMETER, "null signal buffer");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    const size_t xe = (size_t)c->n * b;
    FGB_CUDA(c->x.ensure(xe * c->sig));
    FGB_CUDA(c->y.ensure(xe * c->sig * n_alpha));
    if (int st = upload_signal(c, x, xe, c->x.p)) return st;
    if (int st = apply_device(c, alphas, n_alpha, l_used, inverse != 0, c->x.p, b, c->y.p)) return st;
    return download_signal(c, c->y.p, xe * n_alpha, y);
    FGB_GUARD_END
}

int fgfrft_apply_matrix(const double* q, int64_t n, int inverse, const double* x, int64_t b, double* y, int device) {
    FGB_GUARD_BEGIN
    if (n < 1 || b < 0) return fail(FGFRFT_SHAPE, "apply_forward: signal length does not match operator");
    if (b == 0) return FGFRFT_OK;
    if (!q || !x || !y) return fail(FGFRFT_PARAMETER, "null buffer");
    DeviceGuard dg(device);
    DevBuf dq, dx, dy;
    const size_t qb = (size_t)n * n * 16, xb = (size_t)n * b * 16;
    cudaStream_t st = nullptr;
    FGB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    int rc = FGFRFT_OK;
    do {
        if (dq.ensure(qb) || dx.ensure(xb) || dy.ensure(xb)) {
            rc = fail(FGFRFT_CAPACITY, "device allocation failed");
            break;
        }
        if (cudaMemcpyAsync(dq.p, q, qb, cudaMemcpyHostToDevice, st) ||
            cudaMemcpyAsync(dx.p, x, xb, cudaMemcpyHostToDevice, st)) {
            rc = fail(FGFRFT_CUDA, "upload failed");
            break;
        }
        cudaError_t e = launch_zgemm((int)n, (int)b, (int)n, dq.p, n, 0, inverse != 0, dx.p, n, 0, false, dy.p, n, 0, 1,
                                     false, st);
        if (e != cudaSuccess) {
            rc = fail(FGFRFT_CUDA, std::string("zgemm: ") + cudaGetErrorString(e));
            break;
        }
        g_launches += 1;
        if (cudaMemcpyAsync(y, dy.p, xb, cudaMemcpyDeviceToHost, st) || cudaStreamSynchronize(st)) {
            rc = fail(FGFRFT_CUDA, "download failed");
            break;
        }
    } while (false);
    dq.release();
    dx.release();
    dy.release();
    cudaStreamDestroy(st);
    return rc;
    FGB_GUARD_END
}

int fgfrft_dlda_dev(fgfrft_cache* c, const double* alphas, int n_alpha, const void* g_dev, const void* x_dev,
                    int64_t b, double* s, double* dlda) {
    FGB_GUARD_BEGIN
    if (int st = check_handle(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (b < 0) return fail(FGFRFT_SHAPE, "negative signal count");
    if (!g_dev || !x_dev) return fail(FGFRFT_PARAMETER, "null buffer");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    const size_t width = (size_t)(2 * c->l + 1);
    FGB_CUDA(c->s.ensure((size_t)n_alpha * width * sizeof(double)));
    if (b == 0) {
        FGB_CUDA(cudaMemsetAsync(c->s.p, 0, (size_t)n_alpha * width * sizeof(double), c->stream));
    } else if (c->api_c64 && !tl_internal_signals) {  // complex64 G and X
        const size_t xe = (size_t)c->n * b;
        FGB_CUDA(c->bx.ensure(xe * 16));
        FGB_CUDA(c->by.ensure(xe * n_alpha * 16));
        FGB_LAUNCH(launch_promote(x_dev, c->bx.p, (int64_t)xe, c->stream), 1);
        FGB_LAUNCH(launch_promote(g_dev, c->by.p, (int64_t)(xe * n_alpha), c->stream), 1);
        if (int st = dots_device(c, n_alpha, c->by.p, c->bx.p, b, c->s.as<double>())) return st;
    } else if (int st = dots_device(c, n_alpha, g_dev, x_dev, b, c->s.as<double>())) {
        return st;
    }
    std::vector<double> sh((size_t)n_alpha * width);
    FGB_CUDA(cudaMemcpyAsync(sh.data(), c->s.p, sh.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    std::vector<double> dc(width);
    for (int a = 0; a < n_alpha; ++a) {
        host_sinc_coeffs(alphas[a], c->l, nullptr, dc.data());
        double acc = 0.0;
        for (size_t k = 0; k < width; ++k) acc += dc[k] * sh[a * width + k];
        if (dlda) dlda[a] = acc;
    }
    if (s) std::memcpy(s, sh.data(), sh.size() * sizeof(double));
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_dlda(fgfrft_cache* c, const double* alphas, int n_alpha, const double* g, const double* x, int64_t b,
                double* s, double* dlda) {
    FGB_GUARD_BEGIN
    if (int st = check_handle(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (b < 0) return fail(FGFRFT_SHAPE, "negative signal count");
    if ((!g || !x) && b > 0) return fail(FGFRFT_PARAMETER, "null buffer");
    {
        std::lock_guard<std::mutex> lk(c->mu);
        DeviceGuard dg(c->device);
        const size_t xe = (size_t)c->n * (b > 0 ? b : 1);
        FGB_CUDA(c->x.ensure(xe * c->sig));
        FGB_CUDA(c->g.ensure(xe * c->sig * n_alpha));
        if (b > 0) {
            if (int st = upload_signal(c, x, xe, c->x.p)) return st;
            if (int st = upload_signal(c, g, xe * n_alpha, c->g.p)) return st;
        }
    }
    InternalSignals internal;
    return fgfrft_dlda_dev(c, alphas, n_alpha, c->g.p, c->x.p, b, s, dlda);
    FGB_GUARD_END
}

int fgfrft_mse_step_dev(fgfrft_cache* c, const double* alphas, int n_alpha, const void* x_dev, const void* xc_dev,
                        int64_t b, void* y_dev, void* loss_dev, void* dlda_dev) {
    HostTimer ht_all(5);
    FGB_GUARD_BEGIN
    if (int st = check_handle(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (b < 1) return fail(FGFRFT_SHAPE, "mse_step: need at least one signal");
    if (!x_dev || !xc_dev || !loss_dev || !dlda_dev) return fail(FGFRFT_PARAMETER, "null buffer");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    const int n = (int)c->n;
    const int l = c->l;
    const size_t width = (size_t)(2 * l + 1);
    const size_t blk = (size_t)n * b;
    void* y_c64 = nullptr;
    if (c->api_c64 && !tl_internal_signals) {  // complex64 X, Xc (and Y) at the boundary
        FGB_CUDA(c->bx.ensure(blk * 16));
        FGB_CUDA(c->bxc.ensure(blk * 16));
        FGB_LAUNCH(launch_promote(x_dev, c->bx.p, (int64_t)blk, c->stream), 1);
        FGB_LAUNCH(launch_promote(xc_dev, c->bxc.p, (int64_t)blk, c->stream), 1);
        x_dev = c->bx.p;
        xc_dev = c->bxc.p;
        if (y_dev) {
            FGB_CUDA(c->by.ensure(blk * n_alpha * 16));
            y_c64 = y_dev;
            y_dev = c->by.p;
        }
    }
    struct DemoteY {  // runs on every successful return below
        fgfrft_cache* c;
        void* dst;
        size_t cnt;
        ~DemoteY() {
            if (dst) launch_demote(c->by.p, dst, (int64_t)cnt, c->stream);
        }
    } demote_y{c, y_c64, blk * n_alpha};
    const bool combine = use_power_route(c, n_alpha) && use_int8_combine(c);
    // the node route plans from its own host tables: the exact coefficient tables (bit-identical to
    // sinc.hpp, 2 (2L + 1) libm calls per order) are only evaluated for the routes that consume them
    if (!combine && use_node_route(c, n_alpha, b)) {
        bool ran = false;
        if (int st = mse_node_route(c, alphas, n_alpha, x_dev, xc_dev, b, y_dev, static_cast<double*>(loss_dev),
                                    static_cast<double*>(dlda_dev), true, &ran))
            return st;
        if (ran) return FGFRFT_OK;
    }
    double* coef = nullptr;
    {
        HostTimer ht(0);
        if (int st = upload_coefs(c, alphas, n_alpha, l, &coef)) return st;
    }
    const double* dc_dev = coef + (size_t)n_alpha * width;
    if (combine) {
        FGB_CUDA(c->s.ensure((size_t)n_alpha * width * sizeof(double)));
        return mse_int8_combine(c, coef, dc_dev, n_alpha, x_dev, xc_dev, b, y_dev, static_cast<double*>(loss_dev),
                                c->s.as<double>(), static_cast<double*>(dlda_dev));
    }
    c->last_route = use_power_route(c, n_alpha) ? 1 : 0;
    c->last_nodes = 0;
    if (!use_power_route(c, n_alpha) && n_alpha <= 2 && packed_enabled(c) && use_int8_gemm(c, b) &&
        !use_fused_apply(c, n_alpha, b)) {
        WindowWeights ww;
        const bool win = window_weights(c, alphas, n_alpha, true, c->l, &ww);
        if (win || ensure_step_cache(c))
            return mse_packed_step(c, coef, n_alpha, x_dev, xc_dev, b, y_dev, static_cast<double*>(loss_dev),
                                   static_cast<double*>(dlda_dev), win ? &ww : nullptr);
    }
    if (use_power_route(c, n_alpha)) {
        FGB_CUDA(c->s.ensure((size_t)n_alpha * width * sizeof(double)));
        if (int st = mse_power_route(c, coef, n_alpha, x_dev, xc_dev, b, y_dev, static_cast<double*>(loss_dev),
                                     c->s.as<double>()))
            return st;
        FGB_LAUNCH(launch_coef_dot(dc_dev, c->s.as<double>(), n_alpha, (int)width, static_cast<double*>(dlda_dev),
                                   c->stream),
                   1);
        return FGFRFT_OK;
    }
    const int chunk = alpha_chunk(c, n_alpha);
    const size_t sl = c->mat_elems();
    // One or two orders: synthesise Q and dQ/dalpha together (one pass over the cache, the pair
    // kernel's 2 / 4-order form) and take dL/dalpha = Re<G, dQ X> = Re<G X^H, dQ> as one
    // elementwise dot, instead of a second cache pass for the per-power dots s_k.
    const bool dq_route = n_alpha <= 2 && chunk >= n_alpha && !use_fused_apply(c, n_alpha, b) &&
                          c->dtype == FGFRFT_C128 && std::getenv("FGFRFT_DOTS_ROUTE") == nullptr;
    FGB_CUDA(c->q.ensure((size_t)(dq_route ? 2 : 1) * chunk * sl * c->elem));
    FGB_CUDA(c->g.ensure((size_t)chunk * blk * c->sig));
    FGB_CUDA(c->s.ensure((size_t)n_alpha * width * sizeof(double)));
    FGB_CUDA(c->lpart.ensure(mse_partial_elems(chunk) * sizeof(double)));
    if (!y_dev) FGB_CUDA(c->y.ensure((size_t)chunk * blk * c->sig));
    const double norm = 1.0 / ((double)n * (double)b);
    for (int a0 = 0; a0 < n_alpha; a0 += chunk) {
        const int na = std::min(chunk, n_alpha - a0);
        void* ya = y_dev ? static_cast<char*>(y_dev) + (size_t)a0 * blk * c->sig : c->y.p;
        if (use_fused_apply(c, na, b)) {
            FGB_CUDA(c->partial.ensure(rapply_fused_part_elems(n, na) * sizeof(double)));
            ProfScope ps(KC_SYNTH, c->stream);
            FGB_LAUNCH(launch_rapply_fused(c->slabs, n, l, coef + a0 * width, (int)width, na,
                                           static_cast<const double*>(x_dev), (int)b, c->partial.as<double>(),
                                           static_cast<double*>(ya), c->stream),
                       2);
        } else if (int st = synth_into(c, coef + a0 * width, dq_route ? 2 * na : na, l, c->q.p, true)) {
            return st;  // dq_route: rows [c(a) ..][c'(a) ..] are contiguous in the table (a0 = 0)
        } else if (use_int8_gemm(c, b)) {
            if (int st = int8_qx(c, na, false, c->q.p, x_dev, b, ya)) return st;
        } else {
            ProfScope ps(KC_GEMM, c->stream);
            if (c->real)
                FGB_LAUNCH(launch_rgemm(0, 1, 1, n, 2 * (int)b, n, c->q.p, n, (int64_t)sl, x_dev, n, 0, ya, n,
                                        (int64_t)2 * blk, na, c->stream),
                           1);
            else
                FGB_LAUNCH(gemm(c, n, (int)b, n, c->q.p, n, (int64_t)sl, false, x_dev, n, 0, false, ya, n, (int64_t)blk,
                                na),
                           1);
        }
        if (int st = wait_xc(c)) return st;
        {
            ProfScope ps(KC_ELEMWISE, c->stream);
            FGB_LAUNCH(launch_mse_residual(ya, xc_dev, (int64_t)blk, na, 2.0 * norm, norm, c->g.p,
                                           c->lpart.as<double>(), static_cast<double*>(loss_dev) + a0, c->stream,
                                           (int)c->sig),
                       2);
        }
        if (dq_route) {
            FGB_CUDA(c->m.ensure((size_t)na * sl * c->elem));
            if (int st = gx_device(c, na, c->g.p, x_dev, b)) return st;
            FGB_CUDA(c->partial.ensure((size_t)na * sp_part_elems() * sizeof(double)));
            double* part = c->partial.as<double>();
            const char* dq = c->q.as<char>() + (size_t)na * sl * c->elem;
            ProfScope ps(KC_ELEMWISE, c->stream);
            for (int i = 0; i < na; ++i) {
                const char* mi = c->m.as<char>() + (size_t)i * sl * c->elem;
                if (c->real)
                    FGB_LAUNCH(launch_rdot(reinterpret_cast<const double*>(mi),
                                           reinterpret_cast<const double*>(dq + (size_t)i * sl * c->elem), (int64_t)sl,
                                           part + (size_t)i * sp_part_elems(), c->stream),
                               1);
                else
                    FGB_LAUNCH(launch_cre_dot(mi, dq + (size_t)i * sl * c->elem, false, (int64_t)sl,
                                              part + (size_t)i * sp_part_elems(), c->stream),
                               1);
            }
            FGB_LAUNCH(launch_sum_parts(part, na, 1.0, 1.0, static_cast<double*>(dlda_dev) + a0, c->stream), 1);
            continue;
        }
        if (int st = dots_device(c, na, c->g.p, x_dev, b, c->s.as<double>() + a0 * width)) return st;
    }
    if (!dq_route)
        FGB_LAUNCH(launch_coef_dot(dc_dev, c->s.as<double>(), n_alpha, (int)width, static_cast<double*>(dlda_dev),
                                   c->stream),
                   1);
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_mse_step(fgfrft_cache* c, const double* alphas, int n_alpha, const double* x, const double* xc, int64_t b,
                    double* y, double* loss, double* dlda) {
    FGB_GUARD_BEGIN
    if (int st = check_handle(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (b < 1) return fail(FGFRFT_SHAPE, "mse_step: need at least one signal");
    if (!x || !xc || !loss || !dlda) return fail(FGFRFT_PARAMETER, "null buffer");
    {
        // Packed route (one or two orders, real F, large batch): X goes up in column chunks that
        // overlap the synthesis and the earlier chunks' products, Xc behind it (mse_packed_step).
        std::lock_guard<std::mutex> lk(c->mu);
        DeviceGuard dg(c->device);
        WindowWeights ww;
        bool win = false;
        if (c->dtype == FGFRFT_C128 && !c->api_c64 && n_alpha <= 2 && packed_enabled(c) && use_int8_gemm(c, b) &&
            !use_fused_apply(c, n_alpha, b) && !use_power_route(c, n_alpha) &&
            ((win = window_weights(c, alphas, n_alpha, true, c->l, &ww)) || ensure_step_cache(c))) {
            const size_t xe = (size_t)c->n * b;
            FGB_CUDA(c->x.ensure(xe * 16));
            FGB_CUDA(c->xc.ensure(xe * 16));
            FGB_CUDA(c->loss.ensure((size_t)n_alpha * 2 * sizeof(double)));
            if (y) FGB_CUDA(c->y.ensure(xe * 16 * n_alpha));
            // X onto the link first; the coefficient tables and the step's planning follow behind it
            if (int st = enqueue_host_x(c, x, c->x.p, b)) return st;
            c->xh_pre = x;
            double* coef = nullptr;
            if (int st = upload_coefs(c, alphas, n_alpha, c->l, &coef)) {
                c->xh_pre = nullptr;
                return st;
            }
            double* ld = c->loss.as<double>();
            const int st_step = mse_packed_step(c, coef, n_alpha, c->x.p, c->xc.p, b, y ? c->y.p : nullptr, ld,
                                                ld + n_alpha, win ? &ww : nullptr, x, xc);
            c->xh_pre = nullptr;
            if (st_step) return st_step;
            std::vector<double> out(2 * (size_t)n_alpha);
            FGB_CUDA(cudaMemcpyAsync(out.data(), ld, out.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            if (y) {
                if (int st = download_signal(c, c->y.p, xe * n_alpha, y)) return st;
            }
            FGB_CUDA(cudaStreamSynchronize(c->stream));
            std::memcpy(loss, out.data(), n_alpha * sizeof(double));
            std::memcpy(dlda, out.data() + n_alpha, n_alpha * sizeof(double));
            return FGFRFT_OK;
        }
    }
    {
        std::lock_guard<std::mutex> lk(c->mu);
        DeviceGuard dg(c->device);
        const size_t xe = (size_t)c->n * b;
        FGB_CUDA(c->x.ensure(xe * c->sig));
        FGB_CUDA(c->xc.ensure(xe * c->sig));
        FGB_CUDA(c->loss.ensure((size_t)n_alpha * 2 * sizeof(double)));
        if (y) FGB_CUDA(c->y.ensure(xe * c->sig * n_alpha));
        if (int st = upload_signal(c, x, xe, c->x.p)) return st;
        if (c->dtype == FGFRFT_C128) {
            if (!c->aux_stream) FGB_CUDA(cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking));
            if (!c->xc_evt) FGB_CUDA(cudaEventCreateWithFlags(&c->xc_evt, cudaEventDisableTiming));
            // the side stream must not overwrite Xc while a previous step may still read it
            FGB_CUDA(cudaEventRecord(c->xc_evt, c->stream));
            FGB_CUDA(cudaStreamWaitEvent(c->aux_stream, c->xc_evt, 0));
            FGB_CUDA(cudaMemcpyAsync(c->xc.p, xc, xe * 16, cudaMemcpyHostToDevice, c->aux_stream));
            FGB_CUDA(cudaEventRecord(c->xc_evt, c->aux_stream));
            c->xc_pending = true;
        } else if (int st = upload_signal(c, xc, xe, c->xc.p)) {
            return st;
        }
    }
    double* ld = c->loss.as<double>();
    {
        InternalSignals internal;
        if (int st = fgfrft_mse_step_dev(c, alphas, n_alpha, c->x.p, c->xc.p, b, y ? c->y.p : nullptr, ld,
                                         ld + n_alpha))
            return st;
    }
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    std::vector<double> out(2 * (size_t)n_alpha);
    FGB_CUDA(cudaMemcpyAsync(out.data(), ld, out.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (y) {
        if (int st = download_signal(c, c->y.p, (size_t)c->n * b * n_alpha, y)) return st;
    }
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    std::memcpy(loss, out.data(), n_alpha * sizeof(double));
    std::memcpy(dlda, out.data() + n_alpha, n_alpha * sizeof(double));
    return FGFRFT_OK;
    FGB_GUARD_END
}

}  // extern "C"

// ------------------------------------------------------------------ INT8 tensor-core DGEMM

namespace fgbi {
// Stream-ordered scratch stays in the device pool between calls (no release at sync points).
void keep_pool() {
    static thread_local int done_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (done_dev == dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done_dev = dev;
}
}  // namespace fgbi

int fgfrft_int8_digits(void) { return oz_slices_default(); }

int fgfrft_step_int8_digits(void) { return step_slices(); }

int fgfrft_dgemm_int8_dev(int transa, int transb, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda,
                          const double* b, int64_t ldb, double* c, int64_t ldc, int slices, void* stream) {
    FGB_GUARD_BEGIN
    if (slices == 0) slices = oz_slices_default();
    if (slices < 6 || slices > 8) return fail(FGFRFT_PARAMETER, "slices must be 6, 7 or 8");
    if (m < 1 || n < 1 || k < 1 || k > 16384) return fail(FGFRFT_SHAPE, "dgemm_int8: need m, n >= 1 and 1 <= k <= 16384");
    if (lda < (transa ? k : m) || ldb < (transb ? n : k) || ldc < m)
        return fail(FGFRFT_SHAPE, "dgemm_int8: leading dimension too small");
    if (!a || !b || !c) return fail(FGFRFT_PARAMETER, "null buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    keep_pool();
    const int64_t mp = ceil_div(m, kOzTileA) * kOzTileA, np = ceil_div(n, kOzTileB) * kOzTileB;
    const int64_t kp = ceil_div(k, kOzK) * kOzK;
    const size_t abytes = (size_t)slices * mp * kp, bbytes = (size_t)slices * np * kp;
    const size_t total = abytes + bbytes + (size_t)(mp + np) * (sizeof(int) + sizeof(unsigned long long)) + 256;
    char* ws = nullptr;
    FGB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), total, st));
    int8_t* sa = reinterpret_cast<int8_t*>(ws);
    int8_t* sb = sa + abytes;
    unsigned long long* rmax = reinterpret_cast<unsigned long long*>(sb + bbytes);
    int* ea = reinterpret_cast<int*>(rmax + mp + np);
    int* eb = ea + mp;
    // operand rows: op(A)(r, k) = a[r + k*lda] (or a[k + r*lda]); op(B)^T(r, k) = b[k + r*ldb] (or b[r + k*ldb])
    const OzView va = transa ? OzView{a, lda, 1, 0, 0, 0, (int)m, (int)mp, 1, (int)k, (int)kp, false}
                             : OzView{a, 1, lda, 0, 0, 0, (int)m, (int)mp, 1, (int)k, (int)kp, true};
    const OzView vb = transb ? OzView{b, 1, ldb, 0, 0, 0, (int)n, (int)np, 1, (int)k, (int)kp, true}
                             : OzView{b, ldb, 1, 0, 0, 0, (int)n, (int)np, 1, (int)k, (int)kp, false};
    cudaError_t e;
    {
        ProfScope ps(KC_SLICE, st);
        e = launch_oz_slice(va, slices, kOzTileA, sa, ea, rmax, st);
        if (e == cudaSuccess) e = launch_oz_slice(vb, slices, kOzTileB, sb, eb, rmax + mp, st);
    }
    if (e == cudaSuccess) {
        ProfScope ps(KC_I8GEMM, st);
        e = launch_ozgemm(slices, 0, sa, ea, (int)mp, sb, eb, (int)np, (int)kp, c, ldc, 0, (int)m, (int)mp, (int)n, st);
    }
    cudaFreeAsync(ws, st);
    if (e != cudaSuccess) return fail(FGFRFT_CUDA, std::string("dgemm_int8: ") + cudaGetErrorString(e));
    g_launches += 5;
    return FGFRFT_OK;
    FGB_GUARD_END
}

namespace fgbi {

// Complex product on the INT8 engine: C (m x n, column-major ldc, complex128) = op(A) op(B),
// op 0 = N, 1 = T, 2 = C (conjugate transpose), as ONE real Ozaki GEMM with K doubled:
// A'(r, 2k + e) = (Re, -Im)[e] of op(A)(r, k), B'(2j + c, 2k + e) = [[Re, Im], [Im, -Re]][c][e] of
// op(B)(k, j), so A' B'^T holds (Re C, Im C) in column pairs (2j, 2j + 1) -- the CM 1 epilogue.
int zgemm_int8(int opa, int opb, int64_t m, int64_t n, int64_t k, const void* a, int64_t lda, const void* b,
               int64_t ldb, void* c, int64_t ldc, cudaStream_t st) {
    const int slices = oz_slices_default();
    if (2 * k > 16384) return fail(FGFRFT_SHAPE, "zgemm_int8: k must be <= 8192");
    keep_pool();
    const int64_t mp = ceil_div(m, kOzTileA) * kOzTileA, np = ceil_div(2 * n, kOzTileB) * kOzTileB;
    const int64_t kp = ceil_div(2 * k, kOzK) * kOzK;
    const size_t abytes = (size_t)slices * mp * kp, bbytes = (size_t)slices * np * kp;
    const size_t total = abytes + bbytes + (size_t)(mp + np) * (sizeof(int) + sizeof(unsigned long long)) + 256;
    char* ws = nullptr;
    FGB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), total, st));
    int8_t* sa = reinterpret_cast<int8_t*>(ws);
    int8_t* sb = sa + abytes;
    unsigned long long* rmax = reinterpret_cast<unsigned long long*>(sb + bbytes);
    int* ea = reinterpret_cast<int*>(rmax + mp + np);
    int* eb = ea + mp;
    OzView va{static_cast<const double*>(a), opa == 0 ? 1 : lda, opa == 0 ? lda : 1, 0, 0, opa == 2 ? 1 : 0, (int)m,
              (int)mp, 1, (int)(2 * k), (int)kp, opa == 0};
    va.tiled = 5;
    OzView vb{static_cast<const double*>(b), opb == 0 ? ldb : 1, opb == 0 ? 1 : ldb, 0, 1, opb == 2 ? 1 : 0,
              (int)(2 * n), (int)np, 1, (int)(2 * k), (int)kp, opb != 0};
    vb.tiled = 5;
    cudaError_t e;
    {
        ProfScope ps(KC_SLICE, st);
        e = launch_oz_slice(va, slices, kOzTileA, sa, ea, rmax, st);
        if (e == cudaSuccess) e = launch_oz_slice(vb, slices, kOzTileB, sb, eb, rmax + mp, st);
    }
    if (e == cudaSuccess) {
        ProfScope ps(KC_I8GEMM, st);
        e = launch_ozgemm(slices, 1, sa, ea, (int)mp, sb, eb, (int)np, (int)kp, static_cast<double*>(c), ldc, 0,
                          (int)m, (int)mp, (int)(2 * n), st);
    }
    cudaFreeAsync(ws, st);
    if (e != cudaSuccess) return fail(FGFRFT_CUDA, std::string("zgemm_int8: ") + cudaGetErrorString(e));
    g_launches += 5;
    return FGFRFT_OK;
}

// Complex GEMMs outside a cache handle (spectrum, cascade): the INT8 engine from n = 512 up unless
// FGFRFT_ENGINE=dmma, else DMMA. op as above; batch of independent products with strides.
bool complex_int8_default(int64_t m, int64_t n, int64_t k) {
    static const bool dmma = [] {
        const char* e = std::getenv("FGFRFT_ENGINE");
        return e && !std::strcmp(e, "dmma");
    }();
    return !dmma && m >= 512 && n >= 256 && k >= 512 && k <= 8192;
}

int zgemm_auto(int opa, int opb, int64_t m, int64_t n, int64_t k, const void* a, int64_t lda, int64_t sa,
               const void* b, int64_t ldb, int64_t sb, void* c, int64_t ldc, int64_t sc, int batch, cudaStream_t st) {
    if (opa == 1 || opb == 1) return fail(FGFRFT_PARAMETER, "zgemm_auto: plain transpose not used");
    if (complex_int8_default(m, n, k)) {
        for (int i = 0; i < batch; ++i)
            if (int r = zgemm_int8(opa, opb, m, n, k, static_cast<const double2*>(a) + (size_t)i * sa, lda,
                                   static_cast<const double2*>(b) + (size_t)i * sb, ldb,
                                   static_cast<double2*>(c) + (size_t)i * sc, ldc, st))
                return r;
        return FGFRFT_OK;
    }
    ProfScope ps(KC_GEMM, st);
    FGB_LAUNCH(launch_zgemm((int)m, (int)n, (int)k, a, lda, sa, opa == 2, b, ldb, sb, opb == 2, c, ldc, sc, batch,
                            false, st),
               1);
    return FGFRFT_OK;
}

}  // namespace fgbi

int fgfrft_zgemm_int8_dev(int transa, int transb, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda,
                          const double* b, int64_t ldb, double* c, int64_t ldc, void* stream) {
    FGB_GUARD_BEGIN
    if (transa < 0 || transa > 2 || transb < 0 || transb > 2) return fail(FGFRFT_PARAMETER, "trans must be 0, 1 or 2");
    if (m < 1 || n < 1 || k < 1 || k > 8192) return fail(FGFRFT_SHAPE, "zgemm_int8: need m, n >= 1 and 1 <= k <= 8192");
    if (lda < (transa ? k : m) || ldb < (transb ? n : k) || ldc < m)
        return fail(FGFRFT_SHAPE, "zgemm_int8: leading dimension too small");
    if (!a || !b || !c) return fail(FGFRFT_PARAMETER, "null buffer");
    return zgemm_int8(transa, transb, m, n, k, a, lda, b, ldb, c, ldc, static_cast<cudaStream_t>(stream));
    FGB_GUARD_END
}

