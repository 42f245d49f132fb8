// capi_shard.cu -- row-slab shards (multi-GPU, fgfrft_shard_*), the fused row gather and
// CUDA IPC helpers, and batches of small graphs (fgfrft_batch_*).
#include "capi_internal.cuh"

extern "C" {

// ---------------------------------------------------------------------------- row shards

int fgfrft_shard_create(const double* f, int64_t n, int l, int64_t row_begin, int64_t row_end, uint64_t memory_budget,
                        int device, fgfrft_cache** out) {
    FGB_GUARD_BEGIN
    if (!out) return fail(FGFRFT_PARAMETER, "null output handle pointer");
    *out = nullptr;
    if (l < 1) return fail(FGFRFT_PARAMETER, "PowerCache: truncation order must be >= 1");
    if (n < 1 || !f) return fail(FGFRFT_PARAMETER, "PowerCache: matrix must be non-empty");
    if (row_begin < 0 || row_end > n || row_begin >= row_end || row_begin % kTile != 0 ||
        (row_end % kTile != 0 && row_end != n))
        return fail(FGFRFT_PARAMETER, "shard rows must be [r0, r1) with r0 % 32 == 0 and r1 % 32 == 0 or r1 == n");
    const int64_t rows = row_end - row_begin;
    // real F (graph GFT): real panels, real kernels (as the full cache, learn.hpp:449-451)
    bool real = std::getenv("FGFRFT_NO_REAL") == nullptr;
    for (size_t i = 0; i < (size_t)n * (size_t)n && real; ++i) real = f[2 * i + 1] == 0.0;
    const unsigned __int128 bytes = (unsigned __int128)2 * l * (uint64_t)rows * (uint64_t)n * (real ? 8 : 16);
    if (bytes > memory_budget) {
        std::ostringstream msg;
        msg << "PowerCache shard: " << l << " row and column panels of " << rows << "x" << n << " need "
            << (unsigned long long)bytes << " bytes, over the " << memory_budget << "-byte budget";
        return fail(FGFRFT_CAPACITY, msg.str());
    }
    int ndev = 0;
    FGB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(FGFRFT_PARAMETER, "device index out of range");
    DeviceGuard dg(device);
    auto* c = new fgfrft_cache();
    c->n = n;
    c->l = l;
    c->device = device;
    c->shard = true;
    c->real = real;
    c->elem = real ? 8 : 16;
    c->r0 = row_begin;
    c->r1 = row_end;
    c->fingerprint = host_fnv1a64(f, (size_t)n * (size_t)n * 16);
    const int nI = (int)ceil_div(rows, kTile), nt = (int)ceil_div(n, kTile);
    c->panel_elems = (size_t)nI * nt * kTileElems;
    cudaError_t e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return fail(FGFRFT_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    c->stream = c->own_stream;
    const size_t pbytes = c->panel_elems * c->elem * (size_t)l;
    if (cudaMalloc(&c->slabs, pbytes) != cudaSuccess || cudaMalloc(&c->colp, pbytes) != cudaSuccess) {
        cudaGetLastError();
        destroy_cache(c);
        return fail(FGFRFT_CAPACITY, "PowerCache shard: device allocation failed");
    }
    // Build: Rp_1 = F[R,:], Cp_1 = F[:,R]; Rp_k = Rp_{k-1} F, Cp_k = F Cp_{k-1} (column-major scratch).
    int rc = FGFRFT_OK;
    do {
        const size_t ml = (size_t)n * n, pl = (size_t)rows * n;
        if (c->tmp.ensure((ml + 4 * pl) * 16) != cudaSuccess) {
            rc = fail(FGFRFT_CAPACITY, "PowerCache shard: scratch allocation failed");
            break;
        }
        double2* fb = c->tmp.as<double2>();
        double2 *rp = fb + ml, *rq = rp + pl, *cp = rq + pl, *cq = cp + pl;
        if (cudaMemcpyAsync(fb, f, ml * 16, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
            cudaMemcpy2DAsync(rp, rows * 16, fb + row_begin, n * 16, rows * 16, n, cudaMemcpyDeviceToDevice,
                              c->stream) != cudaSuccess ||
            cudaMemcpyAsync(cp, fb + (size_t)row_begin * n, pl * 16, cudaMemcpyDeviceToDevice, c->stream) !=
                cudaSuccess) {
            rc = fail(FGFRFT_CUDA, "PowerCache shard: staging copies failed");
            break;
        }
        // real: real copies of F and of the panels (8-byte elements) in their own scratch
        DevBuf rs;
        double *fre = nullptr, *rpr = nullptr, *rqr = nullptr, *cpr = nullptr, *cqr = nullptr;
        if (real) {
            if (rs.ensure((ml + 4 * pl) * 8) != cudaSuccess) {
                rc = fail(FGFRFT_CAPACITY, "PowerCache shard: scratch allocation failed");
                break;
            }
            fre = rs.as<double>();
            rpr = fre + ml;
            rqr = rpr + pl;
            cpr = rqr + pl;
            cqr = cpr + pl;
            if (launch_real_part(fb, fre, (int64_t)ml, c->stream) != cudaSuccess ||
                launch_real_part(rp, rpr, (int64_t)pl, c->stream) != cudaSuccess ||
                launch_real_part(cp, cpr, (int64_t)pl, c->stream) != cudaSuccess) {
                rc = fail(FGFRFT_CUDA, "PowerCache shard: real staging failed");
                rs.release();
                break;
            }
        }
        for (int k = 1; k <= l && rc == FGFRFT_OK; ++k) {
            if (k > 1) {
                cudaError_t e1, e2;
                if (real) {
                    e1 = launch_rgemm(0, 0, 0, (int)rows, (int)n, (int)n, rpr, rows, 0, fre, n, 0, rqr, rows, 0, 1,
                                      c->stream);
                    e2 = launch_rgemm(0, 0, 0, (int)n, (int)rows, (int)n, fre, n, 0, cpr, n, 0, cqr, n, 0, 1,
                                      c->stream);
                } else {
                    e1 = launch_zgemm((int)rows, (int)n, (int)n, rp, rows, 0, false, fb, n, 0, false, rq, rows, 0, 1,
                                      false, c->stream);
                    e2 = launch_zgemm((int)n, (int)rows, (int)n, fb, n, 0, false, cp, n, 0, false, cq, n, 0, 1, false,
                                      c->stream);
                }
                if (e1 != cudaSuccess || e2 != cudaSuccess) {
                    rc = fail(FGFRFT_CUDA, "PowerCache shard: panel GEMM failed");
                    break;
                }
                std::swap(rp, rq);
                std::swap(cp, cq);
                std::swap(rpr, rqr);
                std::swap(cpr, cqr);
                g_launches += 2;
            }
            const void* rsrc = real ? static_cast<const void*>(rpr) : static_cast<const void*>(rp);
            const void* csrc = real ? static_cast<const void*>(cpr) : static_cast<const void*>(cp);
            if (launch_rect_to_tiled(rsrc, rows, (int)rows, (int)n,
                                     static_cast<char*>(c->slabs) + (size_t)(k - 1) * c->panel_elems * c->elem,
                                     c->stream, real) != cudaSuccess ||
                launch_rect_to_tiled(csrc, n, (int)n, (int)rows,
                                     static_cast<char*>(c->colp) + (size_t)(k - 1) * c->panel_elems * c->elem,
                                     c->stream, real) != cudaSuccess) {
                rc = fail(FGFRFT_CUDA, "PowerCache shard: tiling failed");
                break;
            }
            g_launches += 2;
        }
        if (rc == FGFRFT_OK && cudaStreamSynchronize(c->stream) != cudaSuccess)
            rc = fail(FGFRFT_CUDA, "PowerCache shard: build failed");
        rs.release();
    } while (false);
    c->tmp.release();
    if (rc != FGFRFT_OK) {
        destroy_cache(c);
        return rc;
    }
    *out = c;
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_shard_destroy(fgfrft_cache* c) {
    FGB_GUARD_BEGIN
    if (c && !c->shard) return fail(FGFRFT_PARAMETER, "not a row-shard handle");
    destroy_cache(c);
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_shard_info(const fgfrft_cache* c, int64_t* n, int* l, int64_t* row_begin, int64_t* row_end,
                      uint64_t* fingerprint) {
    if (int st = check_shard(c)) return st;
    if (n) *n = c->n;
    if (l) *l = c->l;
    if (row_begin) *row_begin = c->r0;
    if (row_end) *row_end = c->r1;
    if (fingerprint) *fingerprint = c->fingerprint;
    return FGFRFT_OK;
}

int fgfrft_shard_set_stream(fgfrft_cache* c, void* stream) {
    if (int st = check_shard(c)) return st;
    std::lock_guard<std::mutex> lk(c->mu);
    c->stream = static_cast<cudaStream_t>(stream);  // NULL = the CUDA default stream
    return FGFRFT_OK;
}

int fgfrft_shard_synthesize_dev(fgfrft_cache* c, const double* alphas, int n_alpha, int which, void* out_dev) {
    FGB_GUARD_BEGIN
    if (int st = check_shard(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (which != FGFRFT_Q && which != FGFRFT_DQ) return fail(FGFRFT_PARAMETER, "which must be FGFRFT_Q or FGFRFT_DQ");
    if (!out_dev) return fail(FGFRFT_PARAMETER, "null output");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    double* coef = nullptr;
    if (int st = upload_coefs(c, alphas, n_alpha, c->l, &coef)) return st;
    const double* table = which == FGFRFT_Q ? coef : coef + (size_t)n_alpha * (2 * c->l + 1);
    ProfScope ps(KC_SYNTH, c->stream);
    FGB_LAUNCH(launch_synth_rows(c->slabs, c->colp, (int)c->n, (int)c->r0, (int)(c->r1 - c->r0), c->l, table, n_alpha,
                                 out_dev, c->stream, c->real, true),
               1);
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_shard_apply_gather_dev(fgfrft_cache* c, const double* alphas, int n_alpha, const void* x_dev, int64_t b,
                                  void* y_full_dev, void* const* peer_y_full, int n_peers) {
    FGB_GUARD_BEGIN
    if (int st = check_shard(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (b < 0) return fail(FGFRFT_SHAPE, "apply_forward: negative signal count");
    if (n_peers < 0 || n_peers > 7 || (n_peers > 0 && !peer_y_full))
        return fail(FGFRFT_PARAMETER, "apply_gather: 0..7 peer buffers");
    if (b == 0) return FGFRFT_OK;
    if (!x_dev || !y_full_dev) return fail(FGFRFT_PARAMETER, "null signal buffer");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    const int n = (int)c->n, rows = (int)(c->r1 - c->r0);
    double* coef = nullptr;
    if (int st = upload_coefs(c, alphas, n_alpha, c->l, &coef)) return st;
    const size_t width = (size_t)(2 * c->l + 1), qs = (size_t)rows * n, blk = (size_t)n * b;
    const int chunk = std::max(1, std::min(n_alpha, (int)(((size_t)4 << 30) / (qs * 16))));
    FGB_CUDA(c->q.ensure((size_t)chunk * qs * 16));
    FGB_CUDA(c->tmp.ensure(8 * sizeof(void*)));  // peer bases as a device array (push kernel)
    const bool i8 = use_int8_gemm(c, b);
    for (int a0 = 0; a0 < n_alpha; a0 += chunk) {
        const int na = std::min(chunk, n_alpha - a0);
        const size_t off = (size_t)a0 * blk + (size_t)c->r0;  // complex elements: order a0, row r0
        double2* yl = static_cast<double2*>(y_full_dev) + off;
        {
            ProfScope ps(KC_SYNTH, c->stream);
            FGB_LAUNCH(launch_synth_rows(c->slabs, c->colp, n, (int)c->r0, rows, c->l, coef + a0 * width, na, c->q.p,
                                         c->stream, c->real, false),
                       1);
        }
        if (i8) {  // rows of Y written locally and into every peer buffer by the GEMM epilogue
            double* pp[7];
            for (int q = 0; q < n_peers; ++q) pp[q] = reinterpret_cast<double*>(static_cast<double2*>(peer_y_full[q]) + off);
            if (int st = int8_qx_gen(c, na, false, c->q.p, rows, rows, (int64_t)qs, x_dev, b, yl, n,
                                     2 * (int64_t)blk, pp, n_peers))
                return st;
            continue;
        }
        {
            ProfScope ps(KC_GEMM, c->stream);
            if (c->real)
                FGB_LAUNCH(launch_rgemm(0, 1, 1, rows, 2 * (int)b, n, c->q.p, rows, (int64_t)qs, x_dev, n, 0, yl, n,
                                        (int64_t)2 * blk, na, c->stream),
                           1);
            else
                FGB_LAUNCH(launch_zgemm(rows, (int)b, n, c->q.p, rows, (int64_t)qs, false, x_dev, n, 0, false, yl, n,
                                        (int64_t)blk, na, false, c->stream),
                           1);
        }
        if (n_peers > 0) {  // DMMA epilogue writes locally: push the rows to the peers (P2P stores)
            std::vector<void*> shifted((size_t)n_peers);
            for (int q = 0; q < n_peers; ++q) shifted[q] = static_cast<double2*>(peer_y_full[q]) + (size_t)a0 * blk;
            FGB_CUDA(cudaMemcpyAsync(c->tmp.p, shifted.data(), (size_t)n_peers * sizeof(void*),
                                     cudaMemcpyHostToDevice, c->stream));
            FGB_LAUNCH(launch_rows_push(static_cast<double2*>(y_full_dev) + (size_t)a0 * blk, n, (int)c->r0, rows,
                                        (int64_t)na * b, c->tmp.as<void*>(), n_peers, c->stream),
                       1);
            FGB_CUDA(cudaStreamSynchronize(c->stream));  // `shifted` is host staging of the copy above
        }
    }
    return FGFRFT_OK;
    FGB_GUARD_END
}

// CUDA IPC of a device buffer for the fused gather: handle (64 bytes) + offset of the pointer in
// its allocation (allocator sub-allocations), and the mapping on a peer process.
int fgfrft_ipc_get(const void* dev_ptr, void* handle_out, uint64_t* offset_out) {
    FGB_GUARD_BEGIN
    if (!dev_ptr || !handle_out || !offset_out) return fail(FGFRFT_PARAMETER, "null argument");
    using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
    static GetRange get_range = [] {
        void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
        return h ? reinterpret_cast<GetRange>(dlsym(h, "cuMemGetAddressRange_v2")) : nullptr;
    }();
    if (!get_range) return fail(FGFRFT_CUDA, "cuMemGetAddressRange unavailable");
    unsigned long long base = 0;
    size_t size = 0;
    if (get_range(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0)
        return fail(FGFRFT_CUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    FGB_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    std::memcpy(handle_out, &h, sizeof h);
    *offset_out = (uint64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_ipc_open(const void* handle, int device, void** base_out) {
    FGB_GUARD_BEGIN
    if (!handle || !base_out) return fail(FGFRFT_PARAMETER, "null argument");
    DeviceGuard dg(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    FGB_CUDA(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_ipc_close(void* base) {
    if (base) cudaIpcCloseMemHandle(base);
    return FGFRFT_OK;
}

int fgfrft_shard_apply_dev(fgfrft_cache* c, const double* alphas, int n_alpha, const void* x_dev, int64_t b,
                           void* y_dev) {
    FGB_GUARD_BEGIN
    if (int st = check_shard(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (b < 0) return fail(FGFRFT_SHAPE, "apply_forward: negative signal count");
    if (b == 0) return FGFRFT_OK;
    if (!x_dev || !y_dev) return fail(FGFRFT_PARAMETER, "null signal buffer");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    const int n = (int)c->n, rows = (int)(c->r1 - c->r0);
    double* coef = nullptr;
    if (int st = upload_coefs(c, alphas, n_alpha, c->l, &coef)) return st;
    const size_t width = (size_t)(2 * c->l + 1), qs = (size_t)rows * n;
    const int chunk = std::max(1, std::min(n_alpha, (int)(((size_t)4 << 30) / (qs * 16))));
    FGB_CUDA(c->q.ensure((size_t)chunk * qs * 16));
    for (int a0 = 0; a0 < n_alpha; a0 += chunk) {
        const int na = std::min(chunk, n_alpha - a0);
        {
            ProfScope ps(KC_SYNTH, c->stream);
            FGB_LAUNCH(launch_synth_rows(c->slabs, c->colp, n, (int)c->r0, rows, c->l, coef + a0 * width, na, c->q.p,
                                         c->stream, c->real, false),
                       1);
        }
        if (use_int8_gemm(c, b)) {
            if (int st = int8_qx_gen(c, na, false, c->q.p, rows, rows, (int64_t)qs, x_dev, b,
                                     static_cast<double2*>(y_dev) + (size_t)a0 * rows * b, rows, 2 * (int64_t)rows * b))
                return st;
            continue;
        }
        ProfScope ps(KC_GEMM, c->stream);
        if (c->real)  // Y[R,:] = Q[R,:] X, real Q rows panel (ld = rows) x complex X
            FGB_LAUNCH(launch_rgemm(0, 1, 1, rows, 2 * (int)b, n, c->q.p, rows, (int64_t)qs, x_dev, n, 0,
                                    static_cast<double2*>(y_dev) + (size_t)a0 * rows * b, rows, (int64_t)2 * rows * b,
                                    na, c->stream),
                       1);
        else
            FGB_LAUNCH(launch_zgemm(rows, (int)b, n, c->q.p, rows, (int64_t)qs, false, x_dev, n, 0, false,
                                    static_cast<double2*>(y_dev) + (size_t)a0 * rows * b, rows, (int64_t)rows * b, na,
                                    false, c->stream),
                       1);
    }
    return FGFRFT_OK;
    FGB_GUARD_END
}

}  // extern "C"

namespace fgbi {

// Row-shard MSE step. s_partial (per-power partials, 2L+1 per order) when requested; otherwise
// dlda_partial = sum_k c'_k s_k directly -- for one or two orders via dQ/dalpha rows synthesised
// in the same cache pass as Q and Re<M[R,:], dQ[R,:]> (no second pass over the panels).
int shard_mse_impl(fgfrft_cache* c, const double* alphas, int n_alpha, const void* x_dev, const void* xc_rows_dev,
                   int64_t b, void* y_rows_dev, void* loss_partial_dev, double* s_partial_dev,
                   double* dlda_partial_dev) {
    const int n = (int)c->n, rows = (int)(c->r1 - c->r0), l = c->l;
    const size_t width = (size_t)(2 * l + 1), qs = (size_t)rows * n, blk = (size_t)rows * b;
    double* coef = nullptr;
    if (int st = upload_coefs(c, alphas, n_alpha, l, &coef)) return st;
    const int chunk = std::max(1, std::min(n_alpha, (int)(((size_t)2 << 30) / (qs * 16))));
    const bool dq_route = !s_partial_dev && n_alpha <= 2 && chunk >= n_alpha &&
                          std::getenv("FGFRFT_DOTS_ROUTE") == nullptr;
    FGB_CUDA(c->q.ensure((size_t)(dq_route ? 2 : 1) * chunk * qs * 16));
    FGB_CUDA(c->m.ensure((size_t)chunk * qs * 16));
    FGB_CUDA(c->g.ensure((size_t)chunk * blk * 16));
    FGB_CUDA(c->lpart.ensure(mse_partial_elems(chunk) * sizeof(double)));
    FGB_CUDA(c->partial.ensure(std::max(dots_rows_partial_elems(n, rows, l, chunk), 2 * sp_part_elems()) *
                               sizeof(double)));
    if (!s_partial_dev && !dq_route) FGB_CUDA(c->s.ensure((size_t)n_alpha * width * sizeof(double)));
    if (!y_rows_dev) FGB_CUDA(c->y.ensure((size_t)chunk * blk * 16));
    const double norm = 1.0 / ((double)n * (double)b);
    const size_t qe = c->real ? 8 : 16;
    for (int a0 = 0; a0 < n_alpha; a0 += chunk) {
        const int na = std::min(chunk, n_alpha - a0);
        double2* ya = y_rows_dev ? static_cast<double2*>(y_rows_dev) + (size_t)a0 * blk : c->y.as<double2>();
        {
            ProfScope ps(KC_SYNTH, c->stream);  // dq_route: table rows [c(a) ..][c'(a) ..] (a0 = 0)
            FGB_LAUNCH(launch_synth_rows(c->slabs, c->colp, n, (int)c->r0, rows, l, coef + a0 * width,
                                         dq_route ? 2 * na : na, c->q.p, c->stream, c->real, false),
                       1);
        }
        if (use_int8_gemm(c, b)) {
            if (int st = int8_qx_gen(c, na, false, c->q.p, rows, rows, (int64_t)qs, x_dev, b, ya, rows,
                                     2 * (int64_t)blk))
                return st;
        } else {
            ProfScope ps(KC_GEMM, c->stream);
            if (c->real)
                FGB_LAUNCH(launch_rgemm(0, 1, 1, rows, 2 * (int)b, n, c->q.p, rows, (int64_t)qs, x_dev, n, 0, ya, rows,
                                        (int64_t)2 * blk, na, c->stream),
                           1);
            else
                FGB_LAUNCH(launch_zgemm(rows, (int)b, n, c->q.p, rows, (int64_t)qs, false, x_dev, n, 0, false, ya, rows,
                                        (int64_t)blk, na, false, c->stream),
                           1);
        }
        {
            ProfScope ps(KC_ELEMWISE, c->stream);
            FGB_LAUNCH(launch_mse_residual(ya, xc_rows_dev, (int64_t)blk, na, 2.0 * norm, 1.0, c->g.p,
                                           c->lpart.as<double>(), static_cast<double*>(loss_partial_dev) + a0,
                                           c->stream, 16),
                       2);
        }
        if (use_int8_gemm(c, b)) {
            if (int st = int8_gx_gen(c, na, c->g.p, rows, x_dev, b, c->m.p, (int64_t)qs)) return st;
        } else {
            ProfScope ps(KC_GEMM, c->stream);  // M[R,:] = G[R,:] X^H (real F: only Re M is needed)
            if (c->real)
                FGB_LAUNCH(launch_rgemm(2, 2, 0, rows, n, 2 * (int)b, c->g.p, rows, (int64_t)2 * blk, x_dev, n, 0, c->m.p,
                                        rows, (int64_t)qs, na, c->stream),
                           1);
            else
                FGB_LAUNCH(launch_zgemm(rows, n, (int)b, c->g.p, rows, (int64_t)blk, false, x_dev, n, 0, true, c->m.p,
                                        rows, (int64_t)qs, na, false, c->stream),
                           1);
        }
        if (dq_route) {  // dlda_partial[a] = Re<M[R,:], dQ[R,:]>
            double* part = c->partial.as<double>();
            const char* dq = c->q.as<char>() + (size_t)na * qs * qe;
            ProfScope ps(KC_ELEMWISE, c->stream);
            for (int i = 0; i < na; ++i) {
                const char* mi = c->m.as<char>() + (size_t)i * qs * qe;
                if (c->real)
                    FGB_LAUNCH(launch_rdot(reinterpret_cast<const double*>(mi),
                                           reinterpret_cast<const double*>(dq + (size_t)i * qs * qe), (int64_t)qs,
                                           part + (size_t)i * sp_part_elems(), c->stream),
                               1);
                else
                    FGB_LAUNCH(launch_cre_dot(mi, dq + (size_t)i * qs * qe, false, (int64_t)qs,
                                              part + (size_t)i * sp_part_elems(), c->stream),
                               1);
            }
            FGB_LAUNCH(launch_sum_parts(part, na, 1.0, 1.0, dlda_partial_dev + a0, c->stream), 1);
            continue;
        }
        double* sp = s_partial_dev ? s_partial_dev : c->s.as<double>();
        ProfScope ps(KC_DOTS, c->stream);
        FGB_LAUNCH(launch_dots_rows(c->slabs, c->colp, n, (int)c->r0, rows, l, c->m.p, (int64_t)qs, na,
                                    c->partial.as<double>(), sp + a0 * width, c->stream, c->real),
                   2);
    }
    if (!s_partial_dev && !dq_route)
        FGB_LAUNCH(launch_coef_dot(coef + (size_t)n_alpha * width, c->s.as<double>(), n_alpha, (int)width,
                                   dlda_partial_dev, c->stream),
                   1);
    return FGFRFT_OK;
}

}  // namespace fgbi

extern "C" {

int fgfrft_shard_mse_partial_dev(fgfrft_cache* c, const double* alphas, int n_alpha, const void* x_dev,
                                 const void* xc_rows_dev, int64_t b, void* y_rows_dev, void* loss_partial_dev,
                                 void* s_partial_dev) {
    FGB_GUARD_BEGIN
    if (int st = check_shard(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (b < 1) return fail(FGFRFT_SHAPE, "mse_step: need at least one signal");
    if (!x_dev || !xc_rows_dev || !loss_partial_dev || !s_partial_dev) return fail(FGFRFT_PARAMETER, "null buffer");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    return shard_mse_impl(c, alphas, n_alpha, x_dev, xc_rows_dev, b, y_rows_dev, loss_partial_dev,
                          static_cast<double*>(s_partial_dev), nullptr);
    FGB_GUARD_END
}

int fgfrft_shard_mse_dlda_partial_dev(fgfrft_cache* c, const double* alphas, int n_alpha, const void* x_dev,
                                      const void* xc_rows_dev, int64_t b, void* y_rows_dev, void* loss_partial_dev,
                                      void* dlda_partial_dev) {
    FGB_GUARD_BEGIN
    if (int st = check_shard(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (b < 1) return fail(FGFRFT_SHAPE, "mse_step: need at least one signal");
    if (!x_dev || !xc_rows_dev || !loss_partial_dev || !dlda_partial_dev) return fail(FGFRFT_PARAMETER, "null buffer");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    return shard_mse_impl(c, alphas, n_alpha, x_dev, xc_rows_dev, b, y_rows_dev, loss_partial_dev, nullptr,
                          static_cast<double*>(dlda_partial_dev));
    FGB_GUARD_END
}

// ---------------------------------------------------------------------------- graph batches

int fgfrft_batch_create(const double* fs, int64_t graphs, int64_t n, int l, int device, fgfrft_cache** out) {
    FGB_GUARD_BEGIN
    if (!out) return fail(FGFRFT_PARAMETER, "null output handle pointer");
    *out = nullptr;
    if (l < 1) return fail(FGFRFT_PARAMETER, "PowerCache: truncation order must be >= 1");
    if (graphs < 1 || graphs > 65535 || !fs) return fail(FGFRFT_PARAMETER, "graph batch: need 1..65535 graphs");
    if (n < 1 || n > batch_max_n()) return fail(FGFRFT_PARAMETER, "graph batch: n must be in 1..64");
    if (l > 255) return fail(FGFRFT_PARAMETER, "graph batch: l must be <= 255");
    int ndev = 0;
    FGB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(FGFRFT_PARAMETER, "device index out of range");
    DeviceGuard dg(device);
    auto* c = new fgfrft_cache();
    c->n = n;
    c->l = l;
    c->device = device;
    c->dtype = FGFRFT_C64;
    c->elem = 8;
    c->graphs = graphs;
    c->fingerprint = host_fnv1a64(fs, (size_t)graphs * n * n * 16);
    if (std::getenv("FGFRFT_NO_REAL") == nullptr) {  // every F real: real float slabs (half the bytes)
        bool real = true;
        for (size_t i = 0; i < (size_t)graphs * n * n && real; ++i) real = fs[2 * i + 1] == 0.0;
        c->real = real;
        if (real) c->elem = 4;
    }
    cudaError_t e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return fail(FGFRFT_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    c->stream = c->own_stream;
    const size_t slab = 4 * (size_t)kTileElems;  // padded 64 x 64
    if (cudaMalloc(&c->slabs, (size_t)graphs * l * slab * c->elem) != cudaSuccess) {
        cudaGetLastError();
        destroy_cache(c);
        return fail(FGFRFT_CAPACITY, "graph batch: device allocation failed");
    }
    int rc = FGFRFT_OK;
    const size_t ml = (size_t)n * n;
    do {
        if (c->tmp.ensure(3 * graphs * ml * 16) != cudaSuccess) {
            rc = fail(FGFRFT_CAPACITY, "graph batch: scratch allocation failed");
            break;
        }
        double2* fb = c->tmp.as<double2>();
        double2* prev = fb + graphs * ml;
        double2* cur = prev + graphs * ml;
        if (cudaMemcpyAsync(fb, fs, graphs * ml * 16, cudaMemcpyHostToDevice, c->stream) != cudaSuccess) {
            rc = fail(FGFRFT_CUDA, "graph batch: upload failed");
            break;
        }
        const double2* p = fb;
        for (int k = 1; k <= l; ++k) {
            if (k > 1) {  // P_k = F P_{k-1} for every graph (batched DMMA GEMM)
                if (launch_zgemm((int)n, (int)n, (int)n, fb, n, (int64_t)ml, false, p, n, (int64_t)ml, false, cur, n,
                                 (int64_t)ml, (int)graphs, false, c->stream) != cudaSuccess) {
                    rc = fail(FGFRFT_CUDA, "graph batch: GEMM failed");
                    break;
                }
                p = cur;
                std::swap(prev, cur);
                g_launches += 1;
            }
            if (launch_batch_to_tiled(p, (int)graphs, (int)n, l, k, c->slabs, c->real, c->stream) != cudaSuccess) {
                rc = fail(FGFRFT_CUDA, "graph batch: tiling failed");
                break;
            }
            g_launches += 1;
        }
        if (rc == FGFRFT_OK && cudaStreamSynchronize(c->stream) != cudaSuccess)
            rc = fail(FGFRFT_CUDA, "graph batch: build failed");
    } while (false);
    c->tmp.release();
    if (rc != FGFRFT_OK) {
        destroy_cache(c);
        return rc;
    }
    *out = c;
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_batch_destroy(fgfrft_cache* c) {
    FGB_GUARD_BEGIN
    if (c && c->graphs <= 0) return fail(FGFRFT_PARAMETER, "not a graph-batch handle");
    destroy_cache(c);
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_batch_set_stream(fgfrft_cache* c, void* stream) {
    if (int st = check_batch(c)) return st;
    std::lock_guard<std::mutex> lk(c->mu);
    c->stream = static_cast<cudaStream_t>(stream);  // NULL = the CUDA default stream
    return FGFRFT_OK;
}

namespace fgbi {
int batch_coefs(fgfrft_cache* c, const double* alphas_dev, int heads, double** coef) {
    const size_t orders = (size_t)c->graphs * heads;
    c->coef_l = -1;  // the host-table memo no longer describes `coef`
    FGB_CUDA(c->coef.ensure(batch_coef_bytes((int)c->graphs, heads, c->l)));
    FGB_LAUNCH(launch_batch_coef(alphas_dev, (int)orders, c->l, c->coef.as<double>(), c->stream, heads), 1);
    *coef = c->coef.as<double>();
    return FGFRFT_OK;
}
}  // namespace fgbi

int fgfrft_batch_forward_dev(fgfrft_cache* c, const double* alphas_dev, int heads, const void* x_dev, int64_t ch,
                             void* y_dev) {
    FGB_GUARD_BEGIN
    if (int st = check_batch(c)) return st;
    if (heads < 1 || heads > batch_max_heads()) return fail(FGFRFT_PARAMETER, "graph batch: heads must be 1..4");
    if (ch < 1 || ch > batch_max_channels()) return fail(FGFRFT_SHAPE, "graph batch: channels must be 1..64");
    if (!alphas_dev || !x_dev || !y_dev) return fail(FGFRFT_PARAMETER, "null buffer");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    double* coef = nullptr;
    if (int st = batch_coefs(c, alphas_dev, heads, &coef)) return st;
    ProfScope ps(KC_SYNTH, c->stream);
    FGB_LAUNCH(launch_batch_forward(c->slabs, (int)c->graphs, (int)c->n, c->l, coef, heads, x_dev, (int)ch, y_dev,
                                    c->real, c->stream),
               1);
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_batch_dlda_dev(fgfrft_cache* c, const double* alphas_dev, int heads, const void* g_dev, const void* x_dev,
                          int64_t ch, void* dlda_dev) {
    FGB_GUARD_BEGIN
    if (int st = check_batch(c)) return st;
    if (heads < 1 || heads > batch_max_heads()) return fail(FGFRFT_PARAMETER, "graph batch: heads must be 1..4");
    if (ch < 1 || ch > batch_max_channels()) return fail(FGFRFT_SHAPE, "graph batch: channels must be 1..64");
    if (!alphas_dev || !g_dev || !x_dev || !dlda_dev) return fail(FGFRFT_PARAMETER, "null buffer");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    double* coef = nullptr;
    if (int st = batch_coefs(c, alphas_dev, heads, &coef)) return st;
    ProfScope ps(KC_DOTS, c->stream);
    FGB_LAUNCH(launch_batch_dlda(c->slabs, (int)c->graphs, (int)c->n, c->l, coef, heads, g_dev, x_dev, (int)ch,
                                 static_cast<double*>(dlda_dev), c->real, c->stream),
               1);
    return FGFRFT_OK;
    FGB_GUARD_END
}

}  // extern "C"
