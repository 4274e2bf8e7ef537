// capi.cpp — the extern "C" boundary (include/svdbgpu.h). Argument checking, error mapping
// (svdb::Errc + 1 / SVDBGPU_E_*), host<->device staging for the host-buffer entry points.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "grid_impl.hpp"
#include "svdbgpu.h"
#include "svdbgpu_internal.hpp"

namespace svdbgpu {

namespace {
thread_local std::string g_error;

const char* errc_name(Errc c)
{
    switch (c) { // errors.hpp:25-39
    case Errc::io_error: return "IoError";
    case Errc::size_mismatch: return "SizeMismatch";
    case Errc::non_finite_voxel: return "NonFiniteVoxel";
    case Errc::out_of_bounds: return "OutOfBounds";
    case Errc::misaligned: return "Misaligned";
    case Errc::empty_box: return "EmptyBox";
    case Errc::invalid_quality: return "InvalidQuality";
    case Errc::bad_magic: return "BadMagic";
    case Errc::version_mismatch: return "VersionMismatch";
    case Errc::corrupt_index: return "CorruptIndex";
    case Errc::dims_mismatch: return "DimsMismatch";
    }
    return "UnknownError";
}
} // namespace

void set_error(const std::string& msg) { g_error = msg; }

int fail(Errc code, const std::string& msg)
{
    g_error = std::string(errc_name(code)) + ": " + msg;
    return int(code) + 1;
}

int fail_code(int code, const std::string& msg)
{
    g_error = msg;
    return code;
}

} // namespace svdbgpu

using namespace svdbgpu;

namespace {

template <typename F>
int guarded(F&& f)
{
    try {
        return f();
    } catch (const std::bad_alloc&) {
        return fail_code(SVDBGPU_E_OOM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail_code(SVDBGPU_E_INVALID_ARG, e.what());
    }
}

// RAII device scratch for the host-buffer entry points.
struct DevBuf {
    void* p = nullptr;
    ~DevBuf() { cudaFree(p); }
};

} // namespace

extern "C" {

int svdbgpu_abi_version(void) { return SVDBGPU_ABI_VERSION; }

const char* svdbgpu_last_error(void) { return g_error.c_str(); }

int svdbgpu_device_count(int32_t* out)
{
    if (!out)
        return fail_code(SVDBGPU_E_INVALID_ARG, "out is null");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    *out = e == cudaSuccess ? n : 0;
    if (e != cudaSuccess) {
        cudaGetLastError();
        return cuda_fail(e, "cudaGetDeviceCount");
    }
    return 0;
}

void svdbgpu_free(void* p) { std::free(p); }

int svdbgpu_grid_create(const uint8_t* svdb, size_t n, int32_t codec, int32_t device, svdbgpu_grid** out)
{
    if (!out)
        return fail_code(SVDBGPU_E_INVALID_ARG, "out is null");
    *out = nullptr;
    return guarded([&] {
        GridImpl* impl = nullptr;
        int rc = grid_create(svdb, n, codec, device, &impl);
        if (rc)
            return rc;
        *out = new svdbgpu_grid{std::unique_ptr<GridImpl>(impl)};
        return 0;
    });
}

int svdbgpu_grid_destroy(svdbgpu_grid* g)
{
    delete g;
    return 0;
}

int svdbgpu_grid_info_get(const svdbgpu_grid* g, svdbgpu_grid_info* o)
{
    if (!g || !o)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null grid/info");
    const GridImpl& G = *g->impl;
    std::memset(o, 0, sizeof *o);
    for (int a = 0; a < 3; ++a)
        o->dims[a] = G.dg.dims[a];
    o->background = G.dg.background;
    o->voxel_type = G.voxel_type;
    o->codec = G.codec;
    o->value_domain[0] = G.value_domain[0];
    o->value_domain[1] = G.value_domain[1];
    o->n_upper = G.n_upper;
    o->n_lower = G.n_lower;
    o->n_leaf = G.n_leaf;
    o->n_root = G.n_root;
    o->svdb_bytes = G.svdb_bytes;
    o->device_bytes = G.device_bytes;
    o->leaf_payload_bytes = G.leaf_payload_bytes;
    o->device = G.device;
    return 0;
}

int svdbgpu_grid_leaf_codes(const svdbgpu_grid* g, uint64_t first, uint64_t count, uint8_t* codes, float* params)
{
    if (!g)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null grid");
    return guarded([&] { return grid_leaf_codes(g->impl.get(), first, count, codes, params); });
}

int svdbgpu_read_voxels_device(const svdbgpu_grid* g, const int32_t* d_ijk, size_t n, float* d_out, void* stream)
{
    if (!g || (n && (!d_ijk || !d_out)))
        return fail_code(SVDBGPU_E_INVALID_ARG, "null argument");
    cudaSetDevice(g->impl->device);
    return read_voxels_device(g->impl.get(), d_ijk, n, d_out, static_cast<cudaStream_t>(stream));
}

int svdbgpu_sample_device(const svdbgpu_grid* g, const double* d_xyz, size_t n, int32_t mode, float* d_out,
                          void* stream)
{
    if (!g || (n && (!d_xyz || !d_out)) || (mode != 0 && mode != 1))
        return fail_code(SVDBGPU_E_INVALID_ARG, "bad argument");
    cudaSetDevice(g->impl->device);
    return sample_device(g->impl.get(), d_xyz, n, mode, d_out, static_cast<cudaStream_t>(stream));
}

int svdbgpu_read_voxels(const svdbgpu_grid* g, const int32_t* ijk, size_t n, float* out)
{
    if (!g || (n && (!ijk || !out)))
        return fail_code(SVDBGPU_E_INVALID_ARG, "null argument");
    if (!n)
        return 0;
    return guarded([&] {
        GridImpl* G = g->impl.get();
        SVDB_CUDA(cudaSetDevice(G->device));
        DevBuf a, b;
        SVDB_CUDA(cudaMalloc(&a.p, n * 12));
        SVDB_CUDA(cudaMalloc(&b.p, n * 4));
        SVDB_CUDA(cudaMemcpyAsync(a.p, ijk, n * 12, cudaMemcpyHostToDevice, G->stream));
        if (int rc = read_voxels_device(G, static_cast<int32_t*>(a.p), n, static_cast<float*>(b.p), G->stream))
            return rc;
        SVDB_CUDA(cudaMemcpyAsync(out, b.p, n * 4, cudaMemcpyDeviceToHost, G->stream));
        SVDB_CUDA(cudaStreamSynchronize(G->stream));
        return 0;
    });
}

int svdbgpu_sample(const svdbgpu_grid* g, const double* xyz, size_t n, int32_t mode, float* out)
{
    if (!g || (n && (!xyz || !out)) || (mode != 0 && mode != 1))
        return fail_code(SVDBGPU_E_INVALID_ARG, "bad argument");
    if (!n)
        return 0;
    return guarded([&] {
        GridImpl* G = g->impl.get();
        SVDB_CUDA(cudaSetDevice(G->device));
        DevBuf a, b;
        SVDB_CUDA(cudaMalloc(&a.p, n * 24));
        SVDB_CUDA(cudaMalloc(&b.p, n * 4));
        SVDB_CUDA(cudaMemcpyAsync(a.p, xyz, n * 24, cudaMemcpyHostToDevice, G->stream));
        if (int rc = sample_device(G, static_cast<double*>(a.p), n, mode, static_cast<float*>(b.p), G->stream))
            return rc;
        SVDB_CUDA(cudaMemcpyAsync(out, b.p, n * 4, cudaMemcpyDeviceToHost, G->stream));
        SVDB_CUDA(cudaStreamSynchronize(G->stream));
        return 0;
    });
}

int svdbgpu_gradient(const svdbgpu_grid* g, const double* xyz, size_t n, double* out)
{
    if (!g || (n && (!xyz || !out)))
        return fail_code(SVDBGPU_E_INVALID_ARG, "bad argument");
    if (!n)
        return 0;
    return guarded([&] {
        GridImpl* G = g->impl.get();
        SVDB_CUDA(cudaSetDevice(G->device));
        DevBuf a, b;
        SVDB_CUDA(cudaMalloc(&a.p, n * 24));
        SVDB_CUDA(cudaMalloc(&b.p, n * 24));
        SVDB_CUDA(cudaMemcpyAsync(a.p, xyz, n * 24, cudaMemcpyHostToDevice, G->stream));
        if (int rc = gradient_device(G, static_cast<double*>(a.p), n, static_cast<double*>(b.p), G->stream))
            return rc;
        SVDB_CUDA(cudaMemcpyAsync(out, b.p, n * 24, cudaMemcpyDeviceToHost, G->stream));
        SVDB_CUDA(cudaStreamSynchronize(G->stream));
        return 0;
    });
}

int svdbgpu_macrocells(svdbgpu_grid* g, const svdbgpu_tf* tf, int32_t* cells3, float* cmin, float* cmax,
                       float* majorant, uint8_t* empty, size_t cap)
{
    if (!g || !cells3)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null argument");
    return guarded([&] {
        GridImpl* G = g->impl.get();
        std::lock_guard<std::mutex> lk(G->mu);
        SVDB_CUDA(cudaSetDevice(G->device));
        if (int rc = G->ensure_ranges(G->stream, nullptr))
            return rc;
        for (int a = 0; a < 3; ++a)
            cells3[a] = G->cells[a];
        size_t nc = size_t(G->cells[0]) * G->cells[1] * G->cells[2];
        if (!cmin || nc > cap)
            return 0; // size query
        SVDB_CUDA(cudaMemcpy(cmin, G->d_cmin, nc * 4, cudaMemcpyDeviceToHost));
        SVDB_CUDA(cudaMemcpy(cmax, G->d_cmax, nc * 4, cudaMemcpyDeviceToHost));
        if (tf && (majorant || empty)) {
            DevTF dtf;
            if (int rc = G->upload_tf(tf, G->stream, &dtf))
                return rc;
            DevBuf e;
            SVDB_CUDA(cudaMalloc(&e.p, nc));
            if (int rc = majorants(G, dtf, G->stream, static_cast<uint8_t*>(e.p)))
                return rc;
            SVDB_CUDA(cudaStreamSynchronize(G->stream));
            if (majorant)
                SVDB_CUDA(cudaMemcpy(majorant, G->d_maj, nc * 4, cudaMemcpyDeviceToHost));
            if (empty)
                SVDB_CUDA(cudaMemcpy(empty, e.p, nc, cudaMemcpyDeviceToHost));
        }
        return 0;
    });
}

int svdbgpu_render_device(svdbgpu_grid* g, const svdbgpu_tf* tf, const svdbgpu_camera* cam,
                          const svdbgpu_settings* s, float* d_out, int32_t packed, void* stream, svdbgpu_stats* stats)
{
    if (!g)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null grid");
    return guarded([&] {
        std::lock_guard<std::mutex> lk(g->impl->mu);
        return render(g->impl.get(), tf, cam, s, d_out, packed, static_cast<cudaStream_t>(stream), stats);
    });
}

int svdbgpu_render(svdbgpu_grid* g, const svdbgpu_tf* tf, const svdbgpu_camera* cam, const svdbgpu_settings* s,
                   float* rgb_out, svdbgpu_stats* stats)
{
    if (!g || !cam || !s || !rgb_out)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null argument");
    return guarded([&] {
        GridImpl* G = g->impl.get();
        std::lock_guard<std::mutex> lk(G->mu);
        SVDB_CUDA(cudaSetDevice(G->device));
        if (cam->width < 1 || cam->height < 1)
            return fail(Errc::size_mismatch, "image size must be positive");
        const int nranks = s->tile_nranks > 0 ? s->tile_nranks : 1;
        if (nranks > 1 && (s->tile_rank < 0 || s->tile_rank >= nranks))
            return fail_code(SVDBGPU_E_INVALID_ARG, "tile_rank out of range");
        const size_t pix = size_t(cam->width) * size_t(cam->height);
        // a rank may own no tiles (small image, many ranks): it renders nothing and succeeds
        const size_t need = (nranks > 1 ? size_t(tiles_for_rank(cam->width, cam->height, s->tile_rank, nranks)) * 256
                                        : pix) * 3 * sizeof(float);
        if (need > G->img_cap || !G->d_img) {
            cudaFree(G->d_img);
            G->d_img = nullptr;
            G->img_cap = 0;
            SVDB_CUDA(cudaMalloc(&G->d_img, need ? need : 4));
            G->img_cap = need;
        }
        if (int rc = render(G, tf, cam, s, G->d_img, nranks > 1 ? 1 : 0, G->stream, stats))
            return rc;
        if (nranks == 1) {
            SVDB_CUDA(cudaMemcpyAsync(rgb_out, G->d_img, pix * 12, cudaMemcpyDeviceToHost, G->stream));
            SVDB_CUDA(cudaStreamSynchronize(G->stream));
            return 0;
        }
        // scatter this rank's packed tiles into the caller's full image
        std::vector<float> packed(need / sizeof(float));
        SVDB_CUDA(cudaMemcpyAsync(packed.data(), G->d_img, need, cudaMemcpyDeviceToHost, G->stream));
        SVDB_CUDA(cudaStreamSynchronize(G->stream));
        const int tiles_x = (cam->width + 15) / 16;
        const int64_t nt = tiles_for_rank(cam->width, cam->height, s->tile_rank, nranks);
        for (int64_t k = 0; k < nt; ++k) {
            int64_t t = k * nranks + s->tile_rank;
            int x0 = int(t % tiles_x) * 16, y0 = int(t / tiles_x) * 16;
            for (int y = 0; y < 16 && y0 + y < cam->height; ++y)
                for (int x = 0; x < 16 && x0 + x < cam->width; ++x)
                    std::memcpy(rgb_out + (size_t(y0 + y) * cam->width + size_t(x0 + x)) * 3,
                                packed.data() + (size_t(k) * 256 + size_t(y) * 16 + size_t(x)) * 3, 12);
        }
        return 0;
    });
}

int64_t svdbgpu_tiles_for_rank(int32_t width, int32_t height, int32_t rank, int32_t nranks)
{
    return tiles_for_rank(width, height, rank, nranks);
}

int svdbgpu_unpack_tiles_device(const float* d_packed, int32_t nranks, int64_t max_tiles, int32_t width,
                                int32_t height, float* d_rgb, void* stream)
{
    if (!d_packed || !d_rgb)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null buffer");
    return unpack_tiles(d_packed, nranks, max_tiles, width, height, d_rgb, static_cast<cudaStream_t>(stream));
}

int svdbgpu_compress(const float* data, const int32_t dims[3], int32_t voxel_type, double quality, int32_t metric,
                     int32_t threads, uint8_t** svdb_out, size_t* n_out, svdbgpu_compress_report* report)
{
    if (!data || !dims || !svdb_out || !n_out)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null argument");
    if (metric < 0 || metric > 2)
        return fail_code(SVDBGPU_E_INVALID_ARG, "metric must be 0..2");
    return guarded([&] {
        HostBuf bytes;
        int rc = compress(data, dims, voxel_type, quality, metric, threads, bytes, report);
        if (rc)
            return rc;
        *n_out = bytes.n;
        *svdb_out = bytes.release();
        return 0;
    });
}

int svdbgpu_compress_stream(svdbgpu_slab_fn fn, void* user, const int32_t dims[3], int32_t voxel_type, double quality,
                            int32_t metric, int32_t device, uint8_t** svdb_out, size_t* n_out,
                            svdbgpu_compress_report* report, double* seconds)
{
    if (!fn || !dims || !svdb_out || !n_out)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null argument");
    return guarded([&] {
        HostBuf bytes;
        if (int rc = stream_compress_callback(fn, user, dims, voxel_type, quality, metric, device, bytes, report,
                                              seconds))
            return rc;
        *n_out = bytes.n;
        *svdb_out = bytes.release();
        return 0;
    });
}

int svdbgpu_synth_compress(int32_t kind, const int32_t dims[3], uint64_t seed, double quality, int32_t metric,
                           int32_t device, uint8_t** svdb_out, size_t* n_out, svdbgpu_compress_report* report,
                           double* seconds)
{
    if (!dims || !svdb_out || !n_out)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null argument");
    return guarded([&] {
        HostBuf bytes;
        if (int rc = stream_compress_synth(kind, dims, seed, quality, metric, device, bytes, report, seconds))
            return rc;
        *n_out = bytes.n;
        *svdb_out = bytes.release();
        return 0;
    });
}

int svdbgpu_quantise(const uint8_t* svdb, size_t n, int32_t codec, int32_t device, uint8_t** out, size_t* n_out)
{
    if (!svdb || !out || !n_out)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null argument");
    return guarded([&] {
        std::vector<uint8_t> bytes;
        int rc = quantise_svdb(svdb, n, codec, device, bytes);
        if (rc)
            return rc;
        auto* p = static_cast<uint8_t*>(std::malloc(bytes.size() ? bytes.size() : 1));
        if (!p)
            return fail_code(SVDBGPU_E_OOM, "host allocation failed");
        std::memcpy(p, bytes.data(), bytes.size());
        *out = p;
        *n_out = bytes.size();
        return 0;
    });
}

int svdbgpu_synth(int32_t kind, const int32_t dims[3], uint64_t seed, int32_t threads, float* out)
{
    if (!dims || !out || kind < 0 || kind > 3)
        return fail_code(SVDBGPU_E_INVALID_ARG, "bad argument");
    return guarded([&] { return synth(kind, dims, seed, threads, out); });
}

} // extern "C"
