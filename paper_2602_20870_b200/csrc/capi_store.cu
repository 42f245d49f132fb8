// capi_store.cu -- the on-disk power cache (fgfrft_cache_save / _load).
#include "capi_internal.cuh"

// ------------------------------------------------------------------ on-disk power cache
//
// the reference rebuilds its cache every run (no binary format for F or the
// powers, io.hpp holds only PGM/XYZ/CSV/manifest). File layout (little endian):
//   CacheFileHeader (128 bytes)
//   F: n x n complex128, column-major -- the bytes content_fingerprint hashes (gft.hpp:46-48)
//   the resident slabs exactly as in HBM (tiled 32 x 32, padded to npad, real / c128 / c64)
//   one u64: order-independent checksum of the slab bytes (store.cu), re-checked after load
// The slabs move through two pinned 64 MiB staging buffers so file IO overlaps the copies.

namespace fgbi {

struct CacheFileHeader {
    char magic[8];  // "FGFRFTC\x01"
    uint32_t version, dtype, real, elem;
    int64_t n;
    int32_t l, tile;
    uint64_t fingerprint, slab_bytes, f_bytes;
    uint64_t reserved[7];
    uint64_t header_fnv;  // fnv1a64 of the preceding 120 bytes
};
static_assert(sizeof(CacheFileHeader) == 128, "cache file header is 128 bytes");
constexpr char kCacheMagic[8] = {'F', 'G', 'F', 'R', 'F', 'T', 'C', 1};
constexpr size_t kStageBytes = (size_t)64 << 20;

struct FileCloser {
    std::FILE* f = nullptr;
    ~FileCloser() {
        if (f) std::fclose(f);
    }
};
struct PinnedPair {
    void* p[2] = {nullptr, nullptr};
    cudaEvent_t e[2] = {nullptr, nullptr};
    cudaError_t init() {
        for (int i = 0; i < 2; ++i) {
            if (cudaError_t r = cudaMallocHost(&p[i], kStageBytes)) return r;
            if (cudaError_t r = cudaEventCreateWithFlags(&e[i], cudaEventDisableTiming)) return r;
        }
        return cudaSuccess;
    }
    ~PinnedPair() {
        for (int i = 0; i < 2; ++i) {
            if (e[i]) cudaEventSynchronize(e[i]), cudaEventDestroy(e[i]);
            if (p[i]) cudaFreeHost(p[i]);
        }
    }
};

int slab_checksum(fgfrft_cache* c, unsigned long long* out) {
    FGB_CUDA(c->lpart.ensure(sizeof(unsigned long long)));
    FGB_LAUNCH(launch_checksum(c->slabs, c->slab_bytes() * (size_t)c->l, c->lpart.as<unsigned long long>(), c->stream),
               1);
    FGB_CUDA(cudaMemcpyAsync(out, c->lpart.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    return FGFRFT_OK;
}

}  // namespace fgbi

extern "C" {

int fgfrft_cache_save(fgfrft_cache* c, const char* path) {
    FGB_GUARD_BEGIN
    if (int st = check_handle(c)) return st;
    if (!path) return fail(FGFRFT_PARAMETER, "null path");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard dg(c->device);
    const size_t ml = c->mat_elems();
    // F = P_1 back in complex128 column-major (the fingerprinted bytes; a complex64 cache stores
    // its rounded F and keeps the original fingerprint in the header)
    std::vector<double> f(2 * ml);
    FGB_CUDA(c->tmp.ensure(ml * 16));
    if (c->real)
        FGB_LAUNCH(launch_rfrom_tiled(c->slab(1), c->tmp.p, (int)c->n, c->stream), 1);
    else
        FGB_LAUNCH(launch_from_tiled(c->slab(1), c->tmp.p, (int)c->n, (int)c->elem, c->stream), 1);
    FGB_CUDA(cudaMemcpyAsync(f.data(), c->tmp.p, ml * 16, cudaMemcpyDeviceToHost, c->stream));
    FGB_CUDA(cudaStreamSynchronize(c->stream));
    c->tmp.release();
    unsigned long long sum = 0;
    if (int st = slab_checksum(c, &sum)) return st;
    CacheFileHeader h{};
    std::memcpy(h.magic, kCacheMagic, 8);
    h.version = 1;
    h.dtype = (uint32_t)(c->api_c64 ? FGFRFT_C64 : c->dtype);
    h.real = c->real ? 1u : 0u;
    h.elem = (uint32_t)c->elem;
    h.n = c->n;
    h.l = c->l;
    h.tile = kTile;
    h.fingerprint = c->fingerprint;
    h.slab_bytes = c->slab_bytes();
    h.f_bytes = ml * 16;
    h.header_fnv = host_fnv1a64(&h, offsetof(CacheFileHeader, header_fnv));
    FileCloser fc;
    fc.f = std::fopen(path, "wb");
    if (!fc.f) return fail(FGFRFT_IO, std::string("cannot open ") + path + " for writing");
    if (std::fwrite(&h, sizeof h, 1, fc.f) != 1 || std::fwrite(f.data(), 16, ml, fc.f) != ml)
        return fail(FGFRFT_IO, std::string("failed writing ") + path);
    // slabs: D2H into one staging buffer while the other is written to the file
    PinnedPair pp;
    FGB_CUDA(pp.init());
    const size_t total = c->slab_bytes() * (size_t)c->l;
    const char* src = static_cast<const char*>(c->slabs);
    size_t sizes[2] = {0, 0};
    auto enqueue = [&](size_t off, int b) -> int {
        sizes[b] = std::min(kStageBytes, total - off);
        FGB_CUDA(cudaMemcpyAsync(pp.p[b], src + off, sizes[b], cudaMemcpyDeviceToHost, c->stream));
        FGB_CUDA(cudaEventRecord(pp.e[b], c->stream));
        return FGFRFT_OK;
    };
    if (int st = enqueue(0, 0)) return st;
    for (size_t off = 0, i = 0; off < total; off += kStageBytes, ++i) {
        const int b = (int)(i & 1);
        FGB_CUDA(cudaEventSynchronize(pp.e[b]));
        if (off + kStageBytes < total)
            if (int st = enqueue(off + kStageBytes, b ^ 1)) return st;
        if (std::fwrite(pp.p[b], 1, sizes[b], fc.f) != sizes[b]) return fail(FGFRFT_IO, std::string("failed writing ") + path);
    }
    const uint64_t s64 = sum;
    if (std::fwrite(&s64, 8, 1, fc.f) != 1) return fail(FGFRFT_IO, std::string("failed writing ") + path);
    if (std::fclose(fc.f) != 0) {
        fc.f = nullptr;
        return fail(FGFRFT_IO, std::string("failed writing ") + path);
    }
    fc.f = nullptr;
    return FGFRFT_OK;
    FGB_GUARD_END
}

int fgfrft_cache_load(const char* path, uint64_t memory_budget, int device, fgfrft_cache** out) {
    FGB_GUARD_BEGIN
    if (!out) return fail(FGFRFT_PARAMETER, "null output handle pointer");
    *out = nullptr;
    if (!path) return fail(FGFRFT_PARAMETER, "null path");
    FileCloser fc;
    fc.f = std::fopen(path, "rb");
    if (!fc.f) return fail(FGFRFT_IO, std::string("cannot open ") + path);
    CacheFileHeader h{};
    if (std::fread(&h, sizeof h, 1, fc.f) != 1) return fail(FGFRFT_PARSE, std::string(path) + ": truncated header");
    if (std::memcmp(h.magic, kCacheMagic, 8) != 0) return fail(FGFRFT_PARSE, std::string(path) + ": not a power-cache file");
    if (h.header_fnv != host_fnv1a64(&h, offsetof(CacheFileHeader, header_fnv)))
        return fail(FGFRFT_PARSE, std::string(path) + ": corrupt header");
    if (h.version != 1 || h.tile != kTile)
        return fail(FGFRFT_PARSE, std::string(path) + ": unsupported cache file version or layout");
    if (h.n < 1 || h.l < 1 || h.f_bytes != (uint64_t)h.n * h.n * 16)
        return fail(FGFRFT_PARSE, std::string(path) + ": inconsistent header");
    const size_t ml = (size_t)h.n * (size_t)h.n;
    std::vector<double> f(2 * ml);
    if (std::fread(f.data(), 16, ml, fc.f) != ml) return fail(FGFRFT_PARSE, std::string(path) + ": truncated matrix");
    fgfrft_cache* c = nullptr;
    if (int st = create_common(f.data(), h.n, h.l, memory_budget, (int)h.dtype, device, out, &c)) return st;
    DeviceGuard dg(device);
    int rc = FGFRFT_OK;
    do {
        if (c->dtype == FGFRFT_C64) c->fingerprint = h.fingerprint;  // F stored rounded to complex64
        if (c->fingerprint != h.fingerprint) {
            rc = fail(FGFRFT_NUMERICAL, std::string(path) + ": fingerprint mismatch, the stored matrix is corrupt");
            break;
        }
        if ((c->real ? 1u : 0u) != h.real || c->elem != h.elem || c->slab_bytes() != h.slab_bytes) {
            rc = fail(FGFRFT_PARSE, std::string(path) + ": slab storage differs from this build (real / element size)");
            break;
        }
        // slabs: file -> staging buffer b while the other buffer's H2D copy runs
        PinnedPair pp;
        if (pp.init() != cudaSuccess) {
            rc = fail(FGFRFT_CAPACITY, "cache load: pinned staging allocation failed");
            break;
        }
        const size_t total = c->slab_bytes() * (size_t)c->l;
        char* dst = static_cast<char*>(c->slabs);
        for (size_t off = 0, i = 0; off < total && rc == FGFRFT_OK; off += kStageBytes, ++i) {
            const int b = (int)(i & 1);
            const size_t sz = std::min(kStageBytes, total - off);
            if (i >= 2 && cudaEventSynchronize(pp.e[b]) != cudaSuccess) rc = fail(FGFRFT_CUDA, "cache load: copy failed");
            else if (std::fread(pp.p[b], 1, sz, fc.f) != sz) rc = fail(FGFRFT_PARSE, std::string(path) + ": truncated slabs");
            else if (cudaMemcpyAsync(dst + off, pp.p[b], sz, cudaMemcpyHostToDevice, c->stream) ||
                     cudaEventRecord(pp.e[b], c->stream))
                rc = fail(FGFRFT_CUDA, "cache load: copy failed");
        }
        if (rc != FGFRFT_OK) break;
        uint64_t want = 0;
        if (std::fread(&want, 8, 1, fc.f) != 1) {
            rc = fail(FGFRFT_PARSE, std::string(path) + ": missing checksum");
            break;
        }
        unsigned long long got = 0;
        if ((rc = slab_checksum(c, &got)) != FGFRFT_OK) break;
        if (got != want) {
            rc = fail(FGFRFT_NUMERICAL, std::string(path) + ": slab checksum mismatch, the stored powers are corrupt");
            break;
        }
        if (c->real) {  // the orthogonality flag of the build (power-product / Gram routes)
            DevBuf t;
            if (t.ensure(ml * 16 + ml * 8) != cudaSuccess) {
                rc = fail(FGFRFT_CAPACITY, "cache load: scratch allocation failed");
                break;
            }
            double* fr = reinterpret_cast<double*>(t.as<double2>() + ml);
            if (cudaMemcpyAsync(t.p, f.data(), ml * 16, cudaMemcpyHostToDevice, c->stream) ||
                launch_real_part(t.p, fr, (int64_t)ml, c->stream))
                rc = fail(FGFRFT_CUDA, "cache load: upload failed");
            else
                rc = check_orthogonal(c, fr, reinterpret_cast<double*>(t.p));
            cudaStreamSynchronize(c->stream);
            t.release();
        }
    } while (false);
    if (rc != FGFRFT_OK) {
        destroy_cache(c);
        return rc;
    }
    *out = c;
    return FGFRFT_OK;
    FGB_GUARD_END
}

}  // extern "C"
