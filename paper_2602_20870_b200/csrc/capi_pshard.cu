// capi_pshard.cu -- the multi-GPU form of the packed step route: an NCCL communicator owned by the
// library (fgfrft_comm_*) and PAIR SHARDS of the packed power cache (fgfrft_pshard_*).
//
// Sharding ("tile-pair ownership {(i,j),(j,i)} with a reduce-scatter of Y"): the
// tile pairs {(I,J),(J,I)}, I <= J, are enumerated I-major; rank g owns the pairs whose smaller
// index I lies in [I_g, I_(g+1)), boundaries chosen so every rank owns ~npairs / G pairs
// (fgfrft_pshard_plan). A rank therefore stores 1/G of the L packed slabs (never the full cache:
// it builds its row and column panels P_k[R, :], P_k[:, R] power by power, R = rows [32 I_g,
// 32 I_(g+1)), and packs its pairs from them), and its synthesised tiles cover exactly two
// rectangles of Q and dQ/da:
//     A = rows R x columns [32 I_g, N)        (q1 of its pairs and q2 of pairs (J, I), J in R)
//     B = rows [32 I_(g+1), N) x columns R     (q2 of its pairs with J beyond R)
// so its partial products are two dense Ozaki GEMMs, Y_g[R] = A X[32 I_g:], Y_g[32 I_(g+1):] =
// B X[R], for [Q; dQ] at once. Sum_g Y_g = Y. The step then needs ONE reduce-scatter of [Y; dY]
// (by signal-column chunks: every rank ends with full rows of its columns), the loss and
// Re<Y - Xc, dY> over its columns, and ONE all-reduce of 2A doubles. No exchange during compute.
#include <nccl.h>

#include "capi_internal.cuh"

// ------------------------------------------------------------------ NCCL (loaded at run time)
namespace {

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclCommInitAll) init_all = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclReduceScatter) reduce_scatter = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

// libnccl.so.2 is opened on first use, so the library loads (and every single-GPU entry point
// works) on hosts without NCCL; a process that already loaded NCCL (e.g. through torch) shares it.
const NcclApi* nccl_api() {
    static NcclApi api;
    static bool ok = [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
#define FGB_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
        FGB_SYM(get_unique_id, "ncclGetUniqueId");
        FGB_SYM(init_rank, "ncclCommInitRank");
        FGB_SYM(init_all, "ncclCommInitAll");
        FGB_SYM(destroy, "ncclCommDestroy");
        FGB_SYM(all_reduce, "ncclAllReduce");
        FGB_SYM(reduce_scatter, "ncclReduceScatter");
        FGB_SYM(broadcast, "ncclBroadcast");
        FGB_SYM(all_gather, "ncclAllGather");
        FGB_SYM(group_start, "ncclGroupStart");
        FGB_SYM(group_end, "ncclGroupEnd");
        FGB_SYM(error_string, "ncclGetErrorString");
#undef FGB_SYM
        return api.get_unique_id && api.init_rank && api.init_all && api.destroy && api.all_reduce &&
               api.reduce_scatter && api.broadcast && api.all_gather && api.group_start && api.group_end && api.error_string;
    }();
    return ok ? &api : nullptr;
}

}  // namespace

struct fgfrft_comm {
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0, device = 0;
};

#define FGB_NCCL(expr)                                                                                   \
    do {                                                                                                 \
        ncclResult_t r_ = (expr);                                                                        \
        if (r_ != ncclSuccess)                                                                           \
            return fail(FGFRFT_NCCL, std::string(#expr) + " failed: " + nccl_api()->error_string(r_));  \
    } while (0)

namespace fgbi {

// Tile-row boundaries I_0 = 0 < ... < I_G = nt: the smallest I_g with pairs_before(I_g) >= g npairs / G.
std::vector<int> pshard_plan(int64_t n, int world) {
    const int64_t nt = ceil_div(n, kTile), npairs = nt * (nt + 1) / 2;
    std::vector<int> b(world + 1, 0);
    b[world] = (int)nt;
    int I = 0;
    for (int g = 1; g < world; ++g) {
        const int64_t target = (npairs * g + world - 1) / world;
        while (I < nt && packed_pairs_before(I, nt) < target) ++I;
        b[g] = std::max(I, b[g - 1]);
    }
    return b;
}

int check_pshard(const fgfrft_cache* c) {
    if (!c) return fail(FGFRFT_PARAMETER, "null pair-shard handle");
    if (!c->pshard) return fail(FGFRFT_PARAMETER, "not a pair-shard handle (fgfrft_pshard_create)");
    return FGFRFT_OK;
}

int pshard_build(fgfrft_cache* c, const double* f_dev_real) {
    const int64_t n = c->n, r0 = (int64_t)c->I0 * kTile, r1 = std::min<int64_t>(n, (int64_t)c->I1 * kTile);
    const int64_t rows = r1 - r0;
    const int64_t local = c->pend - c->pbase;
    if (rows <= 0 || local <= 0) return FGFRFT_OK;  // an empty rank (more ranks than tile rows)
    // row panels [rows x n] (ld rows) and column panels [n x rows] (ld n), current and next
    DevBuf pan;
    FGB_CUDA(pan.ensure((size_t)4 * rows * n * sizeof(double)));
    double* rp = pan.as<double>();
    double* rq = rp + rows * n;
    double* cp = rq + rows * n;
    double* cq = cp + rows * n;
    FGB_CUDA(cudaMemcpy2DAsync(rp, rows * 8, f_dev_real + r0, n * 8, rows * 8, n, cudaMemcpyDeviceToDevice, c->stream));
    FGB_CUDA(cudaMemcpyAsync(cp, f_dev_real + r0 * n, (size_t)rows * n * 8, cudaMemcpyDeviceToDevice, c->stream));
    const bool int8 = n >= 2048;  // as the full cache build: the INT8 chain (7 digits) above n = 2048
    for (int k = 1; k <= c->l; ++k) {
        if (k > 1) {  // P_k[R, :] = P_(k-1)[R, :] F,  P_k[:, R] = F P_(k-1)[:, R]  (powers commute)
            if (int8) {
                if (int st = fgfrft_dgemm_int8_dev(0, 0, rows, n, n, rp, rows, f_dev_real, n, rq, rows, 7, c->stream))
                    return st;
                if (int st = fgfrft_dgemm_int8_dev(0, 0, n, rows, n, f_dev_real, n, cp, n, cq, n, 7, c->stream))
                    return st;
            } else {
                FGB_LAUNCH(launch_rgemm(0, 0, 0, (int)rows, (int)n, (int)n, rp, rows, 0, f_dev_real, n, 0, rq, rows, 0,
                                        1, c->stream),
                           1);
                FGB_LAUNCH(launch_rgemm(0, 0, 0, (int)n, (int)rows, (int)n, f_dev_real, n, 0, cp, n, 0, cq, n, 0, 1,
                                        c->stream),
                           1);
            }
            std::swap(rp, rq);
            std::swap(cp, cq);
        }
        FGB_LAUNCH(launch_pack_pairs_from_panels(rp, rows, cp, n, (int)n, c->I0, (int)c->pbase, (int)local, k - 1,
                                                 c->l, c->pk.p, c->pks.as<double>(), c->stream),
                   1);
    }
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    return FGFRFT_OK;
}

int pshard_create(const double* f, int64_t n, int l, uint64_t budget, int world, int rank, int device,
                  fgfrft_comm* comm, fgfrft_cache** out) {
    if (!out) return fail(FGFRFT_PARAMETER, "null output handle pointer");
    *out = nullptr;
    if (l < 1) return fail(FGFRFT_PARAMETER, "PowerCache: truncation order must be >= 1");
    if (n < 1) return fail(FGFRFT_PARAMETER, "PowerCache: matrix must be non-empty");
    if (world < 1 || rank < 0 || rank >= world) return fail(FGFRFT_PARAMETER, "pair shard: rank out of range");
    const bool have_f = f != nullptr;
    if (!have_f && !(comm && comm->world > 1)) return fail(FGFRFT_PARAMETER, "PowerCache: matrix must be non-empty");
    int ndev = 0;
    FGB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(FGFRFT_PARAMETER, "device index out of range");
    const std::vector<int> plan = pshard_plan(n, world);
    const int64_t nt = ceil_div(n, kTile);
    const int I0 = plan[rank], I1 = plan[rank + 1];
    const int64_t pbase = packed_pairs_before(I0, nt), pend = packed_pairs_before(I1, nt);
    const uint64_t pbytes = packed_bytes_pairs(pend - pbase, l), sbytes = (uint64_t)(pend - pbase) * l * 2 * 8;
    if (pbytes + sbytes > budget) {
        std::ostringstream msg;
        msg << "PowerCache pair shard: " << (pend - pbase) << " packed tile pairs x " << l << " powers need "
            << (unsigned long long)(pbytes + sbytes) << " bytes, over the " << budget << "-byte budget";
        return fail(FGFRFT_CAPACITY, msg.str());
    }
    DeviceGuard dg(device);
    auto* c = new fgfrft_cache();
    c->n = n;
    c->l = l;
    c->device = device;
    c->pshard = true;
    c->real = true;
    c->elem = 8;
    c->budget = budget;
    c->world = world;
    c->rank = rank;
    c->I0 = I0;
    c->I1 = I1;
    c->pbase = pbase;
    c->pend = pend;
    c->comm = comm;
    cudaError_t e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return fail(FGFRFT_CUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    c->stream = c->own_stream;
    int rc = FGFRFT_OK;
    do {
        const size_t ml = (size_t)n * n;
        DevBuf fz, fr;
        if (fz.ensure(ml * 16) != cudaSuccess || fr.ensure(ml * 8) != cudaSuccess ||
            c->pk.ensure(std::max<uint64_t>(pbytes, 16)) != cudaSuccess ||
            c->pks.ensure(std::max<uint64_t>(sbytes, 16)) != cudaSuccess) {
            cudaGetLastError();
            rc = fail(FGFRFT_CAPACITY, "PowerCache pair shard: device allocation failed");
            break;
        }
        if (have_f && cudaMemcpyAsync(fz.p, f, ml * 16, cudaMemcpyHostToDevice, c->stream) != cudaSuccess) {
            rc = fail(FGFRFT_CUDA, "PowerCache pair shard: upload of F failed");
            break;
        }
        if (comm && comm->world > 1) {  // F replicated from rank 0 (the only collective of the build)
            const ncclResult_t r = nccl_api()->broadcast(fz.p, fz.p, ml * 2, ncclFloat64, 0, comm->comm, c->stream);
            if (r != ncclSuccess) {
                rc = fail(FGFRFT_NCCL, std::string("ncclBroadcast(F): ") + nccl_api()->error_string(r));
                break;
            }
        }
        std::vector<double> fh(have_f ? 0 : ml * 2);
        if (!have_f) {
            if (cudaMemcpyAsync(fh.data(), fz.p, ml * 16, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
                cudaStreamSynchronize(c->stream) != cudaSuccess) {
                rc = fail(FGFRFT_CUDA, "PowerCache pair shard: download of the broadcast F failed");
                break;
            }
        }
        const double* fhost = have_f ? f : fh.data();
        c->fingerprint = host_fnv1a64(fhost, ml * 16);
        for (size_t i = 0; i < ml; ++i)
            if (fhost[2 * i + 1] != 0.0) {
                rc = fail(FGFRFT_PARAMETER, "pair shards need a real F (graph GFT); use fgfrft_shard_* for a complex F");
                break;
            }
        if (rc) break;
        if (launch_real_part(fz.p, fr.p, (int64_t)ml, c->stream) != cudaSuccess) {
            rc = fail(FGFRFT_CUDA, "PowerCache pair shard: real staging failed");
            break;
        }
        g_launches += 1;
        fz.release();
        rc = pshard_build(c, fr.as<double>());
    } while (false);
    if (rc != FGFRFT_OK) {
        destroy_cache(c);
        return rc;
    }
    c->pk_state = 1;
    *out = c;
    return FGFRFT_OK;
}

// This rank's partial products into c->pp: `rows` blocks (stride 2 n bpad doubles) of n x bpad
// complex, bpad = world * ceil(b / world); only rows [32 I_g, N) and columns < b are ever written,
// the rest stays zero.
// dest != nullptr: the fused reduce-scatter -- the GEMM epilogue stores each output tile into the
// receive slot (for this rank) of the rank owning its signal-column chunk (ndest owners, cb columns
// each): dest[h] + block * 2 n cb + (row + (j - h cb) n) * 2. Otherwise into c->pp (see above).
int pshard_partial(fgfrft_cache* c, const double* coef, int coef_ld, int rows, const void* x_dev, int64_t b,
                   double* const* dest = nullptr, int ndest = 0, int64_t cb = 0) {
    const int S = oz_slices_default();
    const int64_t n = c->n, mp = pad_rows(n), sl = n * n;
    const int64_t bpad = ceil_div(b, c->world) * c->world, blk = 2 * n * bpad;
    const int64_t r0 = (int64_t)c->I0 * kTile, r1 = std::min<int64_t>(n, (int64_t)c->I1 * kTile);
    const size_t pbytes = (size_t)rows * blk * sizeof(double);
    if (!dest && (c->pp.cap < pbytes || c->pp_b != b || c->pp_rows != rows)) {
        FGB_CUDA(c->pp.ensure(pbytes));
        FGB_CUDA(cudaMemsetAsync(c->pp.p, 0, pbytes, c->stream));
        c->pp_b = b;
        c->pp_rows = rows;
    }
    if (r1 <= r0) return FGFRFT_OK;  // no pairs: a zero partial
    const int64_t bp = ceil_div(2 * b, kOzTileB) * kOzTileB;
    const int64_t rvA = r1 - r0, rpA = pad_rows(rvA), kvA = n - r0, kpA = pad_k(kvA);
    const int64_t rvB = n - r1, rpB = pad_rows(std::max<int64_t>(rvB, 1)), kvB = r1 - r0, kpB = pad_k(kvB);
    const size_t qslA = (size_t)S * rows * rpA * kpA, qslB = rvB > 0 ? (size_t)S * rows * rpB * kpB : 0;
    const size_t xslA = (size_t)S * bp * kpA, xslB = rvB > 0 ? (size_t)S * bp * kpB : 0;
    FGB_CUDA(c->q.ensure((size_t)rows * sl * sizeof(double)));
    FGB_CUDA(c->qsl.ensure(qslA + qslB + xslA + xslB));
    const size_t ex_ints = (size_t)rows * (rpA + rpB) + 2 * (size_t)bp;
    const size_t ex_bytes = ((ex_ints * sizeof(int) + 15) & ~(size_t)15) + (size_t)rows * mp * 8 + 2 * (size_t)bp * 8;
    FGB_CUDA(c->qex.ensure(ex_bytes));
    int* exA = c->qex.as<int>();
    int* exB = exA + rows * rpA;
    int* xeA = exB + rows * rpB;
    int* xeB = xeA + bp;
    unsigned long long* rmax =
        reinterpret_cast<unsigned long long*>(c->qex.as<char>() + ((ex_ints * sizeof(int) + 15) & ~(size_t)15));
    unsigned long long* xrm = rmax + rows * mp;
    int8_t* sA = c->qsl.as<int8_t>();
    int8_t* sB = sA + qslA;
    int8_t* xA = sB + qslB;
    int8_t* xB = xA + xslA;
    double* q = c->q.as<double>();
    FGB_CUDA(cudaMemsetAsync(rmax, 0, (size_t)rows * mp * 8, c->stream));
    {
        ProfScope ps(KC_SYNTH, c->stream);
        FGB_LAUNCH(launch_psynth(c->pk.p, c->pks.as<double>(), (int)n, c->l, c->l, coef, coef_ld, rows, q, sl, rmax, mp,
                                 c->stream, (int)c->pbase, (int)c->pend, 0, (int)c->pbase),
                   1);
    }
    if (int st = wait_xc(c)) return st;  // host-buffer step: X (and Xc) uploaded on the aux stream
    {
        ProfScope ps(KC_SLICE, c->stream);
        OzView va{q + r0 + r0 * n, 1, n, sl, 0, 0, (int)rvA, (int)rpA, rows, (int)kvA, (int)kpA, true};
        va.rmb = mp;
        FGB_LAUNCH(launch_oz_slice_ready(va, S, kOzTileA, sA, exA, rmax + r0, c->stream), 1);
        const OzView vx{static_cast<const double*>(x_dev) + 2 * r0, 2 * n, 2, 0, 1, 0, (int)(2 * b), (int)bp, 1,
                        (int)kvA, (int)kpA, false};
        FGB_LAUNCH(launch_oz_slice(vx, S, kOzTileB, xA, xeA, xrm, c->stream), 1);
        if (rvB > 0) {
            OzView vb{q + r1 + r0 * n, 1, n, sl, 0, 0, (int)rvB, (int)rpB, rows, (int)kvB, (int)kpB, true};
            vb.rmb = mp;
            FGB_LAUNCH(launch_oz_slice_ready(vb, S, kOzTileA, sB, exB, rmax + r1, c->stream), 1);
            const OzView vxb{static_cast<const double*>(x_dev) + 2 * r0, 2 * n, 2, 0, 1, 0, (int)(2 * b), (int)bp, 1,
                             (int)kvB, (int)kpB, false};
            FGB_LAUNCH(launch_oz_slice(vxb, S, kOzTileB, xB, xeB, xrm + bp, c->stream), 1);
        }
    }
    ProfScope ps(KC_I8GEMM, c->stream);
    if (dest) {  // GEMM + reduce-scatter in one kernel: tiles go straight to their owners' slots
        auto launch = [&](const int8_t* sa, const int* ea, int64_t rp, const int8_t* sx, const int* xe, int64_t kp,
                          int64_t row0, int64_t rv) -> int {
            OzOut o;
            o.c = dest[0] + 2 * row0;
            o.ldc = n;
            o.sc = 2 * n * cb;
            o.mv = (int)rv;
            o.mp = (int)rp;
            o.nv = (int)(2 * b);
            o.scw = (int)cb;
            o.ssc = 2 * n * cb;
            o.sld = n;
            for (int h = 0; h < ndest; ++h) o.dest[h] = dest[h] + 2 * row0;
            FGB_LAUNCH(launch_ozgemm_ex(S, 1, sa, ea, (int)(rows * rp), sx, xe, (int)bp, (int)kp, o, c->stream), 1);
            return FGFRFT_OK;
        };
        if (int st = launch(sA, exA, rpA, xA, xeA, kpA, r0, rvA)) return st;
        if (rvB > 0)
            if (int st = launch(sB, exB, rpB, xB, xeB, kpB, r1, rvB)) return st;
        return FGFRFT_OK;
    }
    double* pp = c->pp.as<double>();
    FGB_LAUNCH(launch_ozgemm(S, 1, sA, exA, (int)(rows * rpA), xA, xeA, (int)bp, (int)kpA, pp + 2 * r0, n, blk,
                             (int)rvA, (int)rpA, (int)(2 * b), c->stream),
               1);
    if (rvB > 0)
        FGB_LAUNCH(launch_ozgemm(S, 1, sB, exB, (int)(rows * rpB), xB, xeB, (int)bp, (int)kpB, pp + 2 * r1, n, blk,
                                 (int)rvB, (int)rpB, (int)(2 * b), c->stream),
                   1);
    return FGFRFT_OK;
}

// The receive slots of this rank (world x rows blocks x n x cb complex) and every owner's slot for
// this rank: local for itself, CUDA IPC mappings of the peers' buffers (handles exchanged with one
// ncclAllGather) for the others -- remapped only when the buffer changes.
int pshard_map_slots(fgfrft_cache* c, int rows, int64_t cb) {
    const int G = c->world;
    const int64_t slot = (int64_t)rows * 2 * c->n * cb;  // doubles of one source rank's slot
    const size_t need = (size_t)G * slot * sizeof(double);
    if (c->rb.cap < need) {
        for (void* p : c->rb_open) cudaIpcCloseMemHandle(p);
        c->rb_open.clear();
        c->rb_for = nullptr;
        FGB_CUDA(c->rb.ensure(need));
    }
    c->rb_dest.assign(G, nullptr);
    if (G == 1 || !c->comm) {
        c->rb_dest[0] = c->rb.as<double>();
        return FGFRFT_OK;
    }
    if (c->rb_for != c->rb.p) {
        for (void* p : c->rb_open) cudaIpcCloseMemHandle(p);
        c->rb_open.clear();
        c->rb_peer.assign(G, nullptr);
        cudaIpcMemHandle_t mine;
        FGB_CUDA(cudaIpcGetMemHandle(&mine, c->rb.p));
        DevBuf hb;
        FGB_CUDA(hb.ensure((size_t)G * sizeof(mine)));
        FGB_CUDA(cudaMemcpyAsync(hb.as<char>() + (size_t)c->rank * sizeof(mine), &mine, sizeof(mine),
                                 cudaMemcpyHostToDevice, c->stream));
        FGB_NCCL(nccl_api()->all_gather(hb.as<char>() + (size_t)c->rank * sizeof(mine), hb.p, sizeof(mine), ncclUint8,
                                        c->comm->comm, c->stream));
        std::vector<cudaIpcMemHandle_t> all(G);
        FGB_CUDA(cudaMemcpyAsync(all.data(), hb.p, (size_t)G * sizeof(mine), cudaMemcpyDeviceToHost, c->stream));
        FGB_CUDA(cudaStreamSynchronize(c->stream));
        for (int h = 0; h < G; ++h) {
            if (h == c->rank) {
                c->rb_peer[h] = c->rb.p;
                continue;
            }
            void* p = nullptr;
            FGB_CUDA(cudaIpcOpenMemHandle(&p, all[h], cudaIpcMemLazyEnablePeerAccess));
            c->rb_open.push_back(p);
            c->rb_peer[h] = p;
        }
        c->rb_for = c->rb.p;
    }
    for (int h = 0; h < G; ++h) c->rb_dest[h] = static_cast<double*>(c->rb_peer[h]) + (int64_t)c->rank * slot;
    return FGFRFT_OK;
}

// A stream-ordered barrier across the ranks: an all-reduce of one double.
int pshard_barrier(fgfrft_cache* c) {
    FGB_CUDA(c->bar.ensure(sizeof(double)));
    FGB_NCCL(nccl_api()->all_reduce(c->bar.p, c->bar.p, 1, ncclFloat64, ncclSum, c->comm->comm, c->stream));
    return FGFRFT_OK;
}

}  // namespace fgbi

extern "C" {

// ------------------------------------------------------------------ communicator

int fgfrft_comm_unique_id(void* id_out) {
    FGB_GUARD_BEGIN
    if (!id_out) return fail(FGFRFT_PARAMETER, "null id buffer");
    const NcclApi* api = nccl_api();
    if (!api) return fail(FGFRFT_NCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    FGB_NCCL(api->get_unique_id(&id));
    static_assert(sizeof(ncclUniqueId) == FGFRFT_COMM_ID_BYTES, "NCCL unique id size");
    std::memcpy(id_out, &id, sizeof(id));
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_comm_create(const void* id, int world, int rank, int device, fgfrft_comm** out) {
    FGB_GUARD_BEGIN
    if (!out || !id) return fail(FGFRFT_PARAMETER, "null argument");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return fail(FGFRFT_PARAMETER, "comm: rank out of range");
    const NcclApi* api = nccl_api();
    if (!api) return fail(FGFRFT_NCCL, "libnccl.so.2 could not be loaded");
    int ndev = 0;
    FGB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(FGFRFT_PARAMETER, "device index out of range");
    DeviceGuard dg(device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    auto* c = new fgfrft_comm();
    c->world = world;
    c->rank = rank;
    c->device = device;
    const ncclResult_t r = api->init_rank(&c->comm, world, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        return fail(FGFRFT_NCCL, std::string("ncclCommInitRank: ") + api->error_string(r));
    }
    *out = c;
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_comm_create_all(int ndev, const int* devices, fgfrft_comm** out) {
    FGB_GUARD_BEGIN
    if (!out || !devices || ndev < 1) return fail(FGFRFT_PARAMETER, "comm_create_all: need >= 1 device");
    const NcclApi* api = nccl_api();
    if (!api) return fail(FGFRFT_NCCL, "libnccl.so.2 could not be loaded");
    std::vector<ncclComm_t> cs(ndev);
    FGB_NCCL(api->init_all(cs.data(), ndev, devices));
    for (int i = 0; i < ndev; ++i) {
        out[i] = new fgfrft_comm();
        out[i]->comm = cs[i];
        out[i]->world = ndev;
        out[i]->rank = i;
        out[i]->device = devices[i];
    }
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_comm_destroy(fgfrft_comm* c) {
    FGB_GUARD_BEGIN
    if (!c) return FGFRFT_OK;
    if (c->comm && nccl_api()) nccl_api()->destroy(c->comm);
    delete c;
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_comm_info(const fgfrft_comm* c, int* world, int* rank, int* device) {
    if (!c) return fail(FGFRFT_PARAMETER, "null communicator");
    if (world) *world = c->world;
    if (rank) *rank = c->rank;
    if (device) *device = c->device;
    return FGFRFT_OK;
}

// ------------------------------------------------------------------ pair shards

int fgfrft_pshard_plan(int64_t n, int world, int* tile_rows) {
    FGB_GUARD_BEGIN
    if (n < 1 || world < 1 || !tile_rows) return fail(FGFRFT_PARAMETER, "pshard_plan: need n >= 1, world >= 1");
    const std::vector<int> p = pshard_plan(n, world);
    std::copy(p.begin(), p.end(), tile_rows);
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_pshard_create(const double* f, int64_t n, int l, uint64_t memory_budget, fgfrft_comm* comm,
                         fgfrft_cache** out) {
    FGB_GUARD_BEGIN
    if (!comm) return fail(FGFRFT_PARAMETER, "pshard_create: null communicator");
    return pshard_create(f, n, l, memory_budget, comm->world, comm->rank, comm->device, comm, out);
    FGB_GUARD_END
}

int fgfrft_pshard_create_local(const double* f, int64_t n, int l, uint64_t memory_budget, int world, int rank,
                               int device, fgfrft_cache** out) {
    FGB_GUARD_BEGIN
    return pshard_create(f, n, l, memory_budget, world, rank, device, nullptr, out);
    FGB_GUARD_END
}

int fgfrft_pshard_destroy(fgfrft_cache* c) {
    FGB_GUARD_BEGIN
    if (!c) return FGFRFT_OK;
    if (int st = check_pshard(c)) return st;
    destroy_cache(c);
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_pshard_info(const fgfrft_cache* c, int* world, int* rank, int64_t* pair_begin, int64_t* pair_end,
                       int64_t* row_begin, int64_t* row_end, uint64_t* device_bytes) {
    if (int st = check_pshard(c)) return st;
    if (world) *world = c->world;
    if (rank) *rank = c->rank;
    if (pair_begin) *pair_begin = c->pbase;
    if (pair_end) *pair_end = c->pend;
    if (row_begin) *row_begin = std::min<int64_t>(c->n, (int64_t)c->I0 * kTile);
    if (row_end) *row_end = std::min<int64_t>(c->n, (int64_t)c->I1 * kTile);
    if (device_bytes) *device_bytes = c->pk.cap + c->pks.cap;
    return FGFRFT_OK;
}

int fgfrft_pshard_set_stream(fgfrft_cache* c, void* stream) {
    if (int st = check_pshard(c)) return st;
    std::lock_guard<std::mutex> lk(c->mu);
    c->stream = static_cast<cudaStream_t>(stream);
    return FGFRFT_OK;
}

// Partial products of this rank (no collective): out = rows blocks of n x b complex (stride 2 n b
// doubles): with_dq = 1 -> [Y_g(a_0..); dY_g(a_0..)], 0 -> [Y_g(a_0..)]. Sum over the ranks = Y (dY).
int fgfrft_pshard_partial_dev(fgfrft_cache* c, const double* alphas, int n_alpha, int with_dq, const void* x_dev,
                              int64_t b, void* out_dev) {
    FGB_GUARD_BEGIN
    if (int st = check_pshard(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (b < 1 || !x_dev || !out_dev) return fail(FGFRFT_PARAMETER, "pshard_partial: need X, output and b >= 1");
    const int rows = with_dq ? 2 * n_alpha : n_alpha;
    if (rows != 1 && rows != 2 && rows != 4) return fail(FGFRFT_PARAMETER, "pshard: 1 or 2 orders (4 without dQ)");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    double* coef = nullptr;
    if (int st = upload_coefs(c, alphas, n_alpha, c->l, &coef)) return st;
    if (int st = pshard_partial(c, coef, 2 * c->l + 1, rows, x_dev, b)) return st;
    const int64_t n = c->n, bpad = ceil_div(b, c->world) * c->world;
    for (int r = 0; r < rows; ++r)
        FGB_CUDA(cudaMemcpyAsync(static_cast<double*>(out_dev) + (size_t)r * 2 * n * b,
                                 c->pp.as<double>() + (size_t)r * 2 * n * bpad, (size_t)2 * n * b * 8,
                                 cudaMemcpyDeviceToDevice, c->stream));
    return FGFRFT_OK;
    FGB_GUARD_END
}

// This rank's partial products scattered by signal-column chunk straight from the GEMM epilogue:
// dest[h] = this rank's receive slot in owner h's buffer (rows blocks x n x cb complex, cb =
// ceil(b / ndest)); the fused reduce-scatter's data path without its barriers (tests, custom
// transports). Sum over the source ranks of owner h's slots = columns [h cb, (h+1) cb) of the result.
int fgfrft_pshard_partial_scatter_dev(fgfrft_cache* c, const double* alphas, int n_alpha, int with_dq,
                                      const void* x_dev, int64_t b, void* const* dest, int ndest) {
    FGB_GUARD_BEGIN
    if (int st = check_pshard(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (b < 1 || !x_dev || !dest || ndest < 1 || ndest > 8)
        return fail(FGFRFT_PARAMETER, "pshard_partial_scatter: need X, b >= 1 and 1..8 destinations");
    const int rows = with_dq ? 2 * n_alpha : n_alpha;
    if (rows != 1 && rows != 2 && rows != 4) return fail(FGFRFT_PARAMETER, "pshard: 1 or 2 orders (4 without dQ)");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    double* coef = nullptr;
    if (int st = upload_coefs(c, alphas, n_alpha, c->l, &coef)) return st;
    std::vector<double*> d(ndest);
    for (int h = 0; h < ndest; ++h) d[h] = static_cast<double*>(dest[h]);
    return pshard_partial(c, coef, 2 * c->l + 1, rows, x_dev, b, d.data(), ndest, ceil_div(b, ndest));
    FGB_GUARD_END
}

// The MSE step over the communicator: every rank passes the full X and Xc (device); loss and
// dL/da of every order land on every rank (loss_dev, dlda_dev: n_alpha doubles each).
int fgfrft_pshard_mse_step_dev(fgfrft_cache* c, const double* alphas, int n_alpha, const void* x_dev,
                               const void* xc_dev, int64_t b, void* loss_dev, void* dlda_dev) {
    FGB_GUARD_BEGIN
    if (int st = check_pshard(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (n_alpha > 2) return fail(FGFRFT_PARAMETER, "pshard_mse_step: one or two orders per call");
    if (b < 1 || !x_dev || !xc_dev || !loss_dev || !dlda_dev) return fail(FGFRFT_PARAMETER, "null buffer");
    const bool coll = c->comm && c->world > 1;
    if (c->world > 1 && !c->comm) return fail(FGFRFT_PARAMETER, "pshard_mse_step: a local shard has no communicator");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    double* coef = nullptr;
    if (int st = upload_coefs(c, alphas, n_alpha, c->l, &coef)) return st;
    const int rows = 2 * n_alpha;
    const int64_t n = c->n, bpad = ceil_div(b, c->world) * c->world, cb = bpad / c->world, blk = 2 * n * bpad;
    const int64_t chunk = 2 * n * cb;  // doubles of one rank's column chunk of one block
    static const bool nccl_rs = [] {
        const char* e = std::getenv("FGFRFT_PSHARD_RS");
        return e && !std::strcmp(e, "nccl");
    }();
    if (coll && !nccl_rs && c->world <= 8) {
        // fused: the GEMM epilogue stores every tile into its owner's receive slot over NVLink; a
        // barrier before (the owners are done with the previous step's slots) and after (every
        // rank's tiles have landed), then the owner sums its slots in rank order
        if (int st = pshard_map_slots(c, rows, cb)) return st;
        if (int st = pshard_barrier(c)) return st;
        if (int st = pshard_partial(c, coef, 2 * c->l + 1, rows, x_dev, b, c->rb_dest.data(), c->world, cb))
            return st;
        if (int st = pshard_barrier(c)) return st;
        FGB_CUDA(c->ppc.ensure((size_t)rows * chunk * sizeof(double)));
        {
            ProfScope ps(KC_ELEMWISE, c->stream);
            FGB_LAUNCH(launch_sum_slots(c->rb.as<double>(), c->world, (int64_t)rows * chunk, c->ppc.as<double>(),
                                        c->stream),
                       1);
        }
    } else if (int st = pshard_partial(c, coef, 2 * c->l + 1, rows, x_dev, b)) {
        return st;
    }
    const bool fused = coll && !nccl_rs && c->world <= 8;
    const double* yr = fused ? c->ppc.as<double>() : c->pp.as<double>();  // world 1: the whole (only) chunk
    int64_t ystride = fused ? chunk : blk;
    if (coll && !fused) {  // the NCCL reduce-scatter of [Y; dY] by signal-column chunks
        FGB_CUDA(c->ppc.ensure((size_t)rows * chunk * sizeof(double)));
        const NcclApi* api = nccl_api();
        FGB_NCCL(api->group_start());
        for (int r = 0; r < rows; ++r)
            FGB_NCCL(api->reduce_scatter(c->pp.as<double>() + (size_t)r * blk, c->ppc.as<double>() + (size_t)r * chunk,
                                         (size_t)chunk, ncclFloat64, ncclSum, c->comm->comm, c->stream));
        FGB_NCCL(api->group_end());
        yr = c->ppc.as<double>();
        ystride = chunk;
    }
    const int64_t j0 = coll ? c->rank * cb : 0;
    const int64_t valid = std::max<int64_t>(0, std::min<int64_t>(coll ? cb : b, b - j0));
    FGB_CUDA(c->lpart.ensure(mse_dy_part_elems() * sizeof(double)));
    FGB_CUDA(c->loss.ensure((size_t)2 * n_alpha * sizeof(double)));
    double* lb = c->loss.as<double>();
    const double norm = 1.0 / ((double)n * (double)b);
    {
        ProfScope ps(KC_ELEMWISE, c->stream);
        for (int a = 0; a < n_alpha; ++a)
            FGB_LAUNCH(launch_mse_dy(yr + (size_t)a * ystride, yr + (size_t)(n_alpha + a) * ystride,
                                     static_cast<const double*>(xc_dev) + j0 * 2 * n, n * valid, nullptr,
                                     c->lpart.as<double>(), norm, lb + a, lb + n_alpha + a, c->stream),
                       2);
    }
    if (coll) FGB_NCCL(nccl_api()->all_reduce(lb, lb, 2 * (size_t)n_alpha, ncclFloat64, ncclSum, c->comm->comm,
                                              c->stream));
    FGB_CUDA(cudaMemcpyAsync(loss_dev, lb, n_alpha * 8, cudaMemcpyDeviceToDevice, c->stream));
    FGB_CUDA(cudaMemcpyAsync(dlda_dev, lb + n_alpha, n_alpha * 8, cudaMemcpyDeviceToDevice, c->stream));
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_pshard_mse_step(fgfrft_cache* c, const double* alphas, int n_alpha, const double* x, const double* xc,
                           int64_t b, double* loss, double* dlda) {
    FGB_GUARD_BEGIN
    if (int st = check_pshard(c)) return st;
    if (b < 1 || !x || !xc || !loss || !dlda || n_alpha < 1) return fail(FGFRFT_PARAMETER, "null buffer");
    {
        std::lock_guard<std::mutex> lk(c->mu);
        DeviceGuard dg(c->device);
        const size_t xe = (size_t)c->n * b;
        FGB_CUDA(c->x.ensure(xe * 16));
        FGB_CUDA(c->xc.ensure(xe * 16));
        FGB_CUDA(c->dlda.ensure((size_t)2 * n_alpha * 8));
        // X and Xc go up on the aux stream while the synthesis runs (it does not need them); the
        // partial products wait for X right before its slicing, the loss pass for Xc (x_evt).
        if (!c->aux_stream) FGB_CUDA(cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking));
        if (!c->xc_evt) FGB_CUDA(cudaEventCreateWithFlags(&c->xc_evt, cudaEventDisableTiming));
        if (!c->pk_e0) FGB_CUDA(cudaEventCreateWithFlags(&c->pk_e0, cudaEventDisableTiming));
        FGB_CUDA(cudaEventRecord(c->pk_e0, c->stream));  // the previous call's readers are done
        FGB_CUDA(cudaStreamWaitEvent(c->aux_stream, c->pk_e0, 0));
        FGB_CUDA(cudaMemcpyAsync(c->x.p, x, xe * 16, cudaMemcpyHostToDevice, c->aux_stream));
        FGB_CUDA(cudaMemcpyAsync(c->xc.p, xc, xe * 16, cudaMemcpyHostToDevice, c->aux_stream));
        FGB_CUDA(cudaEventRecord(c->xc_evt, c->aux_stream));
        c->xc_pending = true;
    }
    double* out = c->dlda.as<double>();
    if (int st = fgfrft_pshard_mse_step_dev(c, alphas, n_alpha, c->x.p, c->xc.p, b, out, out + n_alpha)) return st;
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    std::vector<double> h(2 * (size_t)n_alpha);
    FGB_CUDA(cudaMemcpyAsync(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    std::memcpy(loss, h.data(), n_alpha * 8);
    std::memcpy(dlda, h.data() + n_alpha, n_alpha * 8);
    return FGFRFT_OK;
    FGB_GUARD_END
}

// Y = F^a X (inverse: Q(-a) X) for 1, 2 or 4 orders, the full Y on every rank (all-reduce of the
// partial products). y_dev: n_alpha blocks of n x b complex.
int fgfrft_pshard_apply_dev(fgfrft_cache* c, const double* alphas, int n_alpha, int inverse, const void* x_dev,
                            int64_t b, void* y_dev) {
    FGB_GUARD_BEGIN
    if (int st = check_pshard(c)) return st;
    if (int st = check_alphas(alphas, n_alpha)) return st;
    if (n_alpha != 1 && n_alpha != 2 && n_alpha != 4) return fail(FGFRFT_PARAMETER, "pshard_apply: 1, 2 or 4 orders");
    if (b < 1 || !x_dev || !y_dev) return fail(FGFRFT_PARAMETER, "null buffer");
    if (c->world > 1 && !c->comm) return fail(FGFRFT_PARAMETER, "pshard_apply: a local shard has no communicator");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    std::vector<double> al(alphas, alphas + n_alpha);
    if (inverse)
        for (double& v : al) v = -v;  // Q(a)^T = Q(-a) bit-exactly (sinc.hpp coefficient mirror)
    double* coef = nullptr;
    if (int st = upload_coefs(c, al.data(), n_alpha, c->l, &coef)) return st;
    if (int st = pshard_partial(c, coef, 2 * c->l + 1, n_alpha, x_dev, b)) return st;
    const int64_t n = c->n, bpad = ceil_div(b, c->world) * c->world;
    for (int r = 0; r < n_alpha; ++r) {
        const double* src = c->pp.as<double>() + (size_t)r * 2 * n * bpad;
        double* dst = static_cast<double*>(y_dev) + (size_t)r * 2 * n * b;
        if (c->comm && c->world > 1)
            FGB_NCCL(nccl_api()->all_reduce(src, dst, (size_t)2 * n * b, ncclFloat64, ncclSum, c->comm->comm,
                                            c->stream));
        else
            FGB_CUDA(cudaMemcpyAsync(dst, src, (size_t)2 * n * b * 8, cudaMemcpyDeviceToDevice, c->stream));
    }
    return FGFRFT_OK;
    FGB_GUARD_END
}

}  // extern "C"
