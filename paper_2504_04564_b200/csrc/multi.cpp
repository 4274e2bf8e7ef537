// multi.cpp — svdbgpu_render_multi: one frame over several devices from one host process
// (SURVEY.md §8b "ndev, devs" / §8e). The reference parallelises render_field's 16x16 tiles over
// host threads (render.hpp:289-313); here every device owns the interleaved tiles t % ndev == k of
// the frame and renders them into a packed buffer, ONE NCCL gather (grouped ncclSend/ncclRecv over
// NVLink / NVSwitch) brings the packed buffers to the first device, k_unpack un-interleaves them and
// the frame is copied to the caller's host image. Paths are keyed per (pixel, sample), so the frame
// is bit-identical to the single-device render for any device count.
//
// NCCL is resolved at first use with dlopen("libnccl.so.2") (RTLD_NOLOAD first, so a process that
// already carries torch's NCCL reuses it): libsvdbgpu.so has no link-time NCCL dependency, and a
// multi-device call without NCCL fails loudly with SVDBGPU_E_NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "grid_impl.hpp"
#include "svdbgpu.h"

namespace svdbgpu {
namespace {

struct Nccl {
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    ncclResult_t (*get_version)(int*) = nullptr;
    std::string why;
    bool ok = false;
};

const Nccl& nccl()
{
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h)
            h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h)
            h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            n.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            return fn != nullptr;
        };
        n.ok = sym(n.comm_init_all, "ncclCommInitAll") && sym(n.group_start, "ncclGroupStart") &&
               sym(n.group_end, "ncclGroupEnd") && sym(n.send, "ncclSend") && sym(n.recv, "ncclRecv") &&
               sym(n.error_string, "ncclGetErrorString") && sym(n.get_version, "ncclGetVersion");
        if (!n.ok)
            n.why = "libnccl.so.2 lacks ncclSend/ncclRecv/ncclCommInitAll";
    });
    return n;
}

int nccl_fail(ncclResult_t r, const char* what)
{
    return fail_code(SVDBGPU_E_NCCL, std::string(what) + ": " + nccl().error_string(r));
}

// One communicator clique per device list, created once with ncclCommInitAll and kept for the life
// of the process (frames re-render on the same devices).
std::mutex g_comm_mu;
std::map<std::vector<int>, std::vector<ncclComm_t>> g_comms;

int comms_for(const std::vector<int>& devs, std::vector<ncclComm_t>& out)
{
    std::lock_guard<std::mutex> lk(g_comm_mu);
    auto it = g_comms.find(devs);
    if (it == g_comms.end()) {
        std::vector<ncclComm_t> c(devs.size());
        ncclResult_t r = nccl().comm_init_all(c.data(), int(devs.size()), devs.data());
        if (r != ncclSuccess)
            return nccl_fail(r, "ncclCommInitAll");
        it = g_comms.emplace(devs, std::move(c)).first;
    }
    out = it->second;
    return 0;
}

int ensure(float*& p, size_t& cap, size_t bytes)
{
    if (bytes <= cap && p)
        return 0;
    cudaFree(p);
    p = nullptr;
    cap = 0;
    SVDB_CUDA(cudaMalloc(&p, bytes ? bytes : 4));
    cap = bytes;
    return 0;
}

} // namespace
} // namespace svdbgpu

using namespace svdbgpu;

extern "C" int svdbgpu_render_multi(svdbgpu_grid* const* grids, int32_t ndev, const svdbgpu_tf* tf,
                                    const svdbgpu_camera* cam, const svdbgpu_settings* s, float* rgb_out,
                                    svdbgpu_stats* stats, double* gather_ms)
{
    if (!grids || ndev < 1 || !cam || !s || !rgb_out)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null argument or ndev < 1");
    if (s->tile_nranks > 1)
        return fail_code(SVDBGPU_E_INVALID_ARG, "svdbgpu_render_multi splits the frame itself (tile_nranks must be 0/1)");
    if (cam->width < 1 || cam->height < 1)
        return fail(Errc::size_mismatch, "image size must be positive");
    std::vector<GridImpl*> G(static_cast<size_t>(ndev));
    std::vector<int> devs(static_cast<size_t>(ndev));
    for (int k = 0; k < ndev; ++k) {
        if (!grids[k])
            return fail_code(SVDBGPU_E_INVALID_ARG, "null grid");
        G[size_t(k)] = grids[k]->impl.get();
        devs[size_t(k)] = G[size_t(k)]->device;
        for (int j = 0; j < 3; ++j)
            if (G[size_t(k)]->dg.dims[j] != G[0]->dg.dims[j])
                return fail(Errc::dims_mismatch, "svdbgpu_render_multi: grids differ in dims");
    }
    {
        std::vector<int> sorted = devs;
        std::sort(sorted.begin(), sorted.end());
        if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
            return fail_code(SVDBGPU_E_INVALID_ARG, "svdbgpu_render_multi: each grid must live on a distinct device");
    }
    try {
        if (gather_ms)
            *gather_ms = 0.0;
        std::vector<ncclComm_t> comms;
        if (ndev > 1) {
            if (!nccl().ok)
                return fail_code(SVDBGPU_E_NCCL, nccl().why);
            if (int rc = comms_for(devs, comms))
                return rc;
        }
        // lock every grid in device-list order (a fixed order: no lock-order inversion between callers)
        std::vector<std::unique_lock<std::mutex>> locks;
        for (int k = 0; k < ndev; ++k)
            locks.emplace_back(G[size_t(k)]->mu);
        const int64_t max_tiles = tiles_for_rank(cam->width, cam->height, 0, ndev);
        const size_t slot = size_t(max_tiles) * 256 * 3; // floats per device slot
        GridImpl* g0 = G[0];
        SVDB_CUDA(cudaSetDevice(g0->device));
        if (int rc = ensure(g0->d_gather, g0->gather_cap, slot * size_t(ndev) * sizeof(float)))
            return rc;
        if (int rc = ensure(g0->d_img, g0->img_cap, size_t(cam->width) * size_t(cam->height) * 12))
            return rc;
        for (int k = 1; k < ndev; ++k) {
            SVDB_CUDA(cudaSetDevice(G[size_t(k)]->device));
            if (int rc = ensure(G[size_t(k)]->d_img, G[size_t(k)]->img_cap, slot * sizeof(float)))
                return rc;
        }
        // 1. every device renders its tiles concurrently (one host thread each: render() waits on
        //    its own stream for the stats); device 0 writes straight into slot 0 of the gather buffer
        std::vector<svdbgpu_stats> st(static_cast<size_t>(ndev));
        std::vector<int> rcs(static_cast<size_t>(ndev), 0);
        std::vector<std::string> errs(static_cast<size_t>(ndev));
        auto work = [&](int k) {
            svdbgpu_settings sk = *s;
            sk.tile_rank = k;
            sk.tile_nranks = ndev;
            GridImpl* g = G[size_t(k)];
            float* out = k == 0 ? g0->d_gather : g->d_img;
            rcs[size_t(k)] = render(g, tf, cam, &sk, out, 1, g->stream, &st[size_t(k)]);
            if (rcs[size_t(k)])
                errs[size_t(k)] = svdbgpu_last_error();
        };
        if (ndev == 1) {
            work(0);
        } else {
            std::vector<std::thread> th;
            for (int k = 0; k < ndev; ++k)
                th.emplace_back(work, k);
            for (auto& t : th)
                t.join();
        }
        for (int k = 0; k < ndev; ++k)
            if (rcs[size_t(k)])
                return fail_code(rcs[size_t(k)], "device " + std::to_string(devs[size_t(k)]) + ": " + errs[size_t(k)]);
        // 2. the one collective: packed tiles of devices 1..n-1 -> slots 1..n-1 on device 0
        NvtxRange nvtx("svdbgpu_render_multi NCCL gather");
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        SVDB_CUDA(cudaSetDevice(g0->device));
        SVDB_CUDA(cudaEventCreate(&e0));
        SVDB_CUDA(cudaEventCreate(&e1));
        SVDB_CUDA(cudaEventRecord(e0, g0->stream));
        if (ndev > 1) {
            const Nccl& N = nccl();
            ncclResult_t r = N.group_start();
            for (int k = 1; k < ndev && r == ncclSuccess; ++k) {
                r = N.send(G[size_t(k)]->d_img, slot, ncclFloat32, 0, comms[size_t(k)], G[size_t(k)]->stream);
                if (r == ncclSuccess)
                    r = N.recv(g0->d_gather + slot * size_t(k), slot, ncclFloat32, k, comms[0], g0->stream);
            }
            ncclResult_t r2 = N.group_end();
            if (r != ncclSuccess || r2 != ncclSuccess) {
                cudaEventDestroy(e0);
                cudaEventDestroy(e1);
                return nccl_fail(r != ncclSuccess ? r : r2, "ncclSend/ncclRecv gather");
            }
        }
        SVDB_CUDA(cudaEventRecord(e1, g0->stream));
        // 3. un-interleave on device 0 and copy the frame out
        if (int rc = unpack_tiles(g0->d_gather, ndev, max_tiles, cam->width, cam->height, g0->d_img, g0->stream))
            return rc;
        SVDB_CUDA(cudaMemcpyAsync(rgb_out, g0->d_img, size_t(cam->width) * size_t(cam->height) * 12,
                                  cudaMemcpyDeviceToHost, g0->stream));
        for (int k = 1; k < ndev; ++k) {
            SVDB_CUDA(cudaSetDevice(G[size_t(k)]->device));
            SVDB_CUDA(cudaStreamSynchronize(G[size_t(k)]->stream));
        }
        SVDB_CUDA(cudaSetDevice(g0->device));
        SVDB_CUDA(cudaStreamSynchronize(g0->stream));
        float gms = 0.0f;
        if (ndev > 1)
            cudaEventElapsedTime(&gms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (gather_ms)
            *gather_ms = gms;
        if (stats) {
            svdbgpu_stats a{};
            for (const auto& x : st) {
                a.paths += x.paths;
                a.samples += x.samples;
                a.lookups += x.lookups;
                a.render_ms = std::max(a.render_ms, x.render_ms);
                a.macrocell_ms = std::max(a.macrocell_ms, x.macrocell_ms);
                a.launches += x.launches;
            }
            a.launches += 1; // k_unpack
            *stats = a;
        }
        return 0;
    } catch (const std::bad_alloc&) {
        return fail_code(SVDBGPU_E_OOM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail_code(SVDBGPU_E_INVALID_ARG, e.what());
    }
}

extern "C" int svdbgpu_nccl_version(int32_t* out)
{
    if (!out)
        return fail_code(SVDBGPU_E_INVALID_ARG, "null argument");
    *out = 0;
    if (!nccl().ok)
        return fail_code(SVDBGPU_E_NCCL, nccl().why);
    int v = 0;
    ncclResult_t r = nccl().get_version(&v);
    if (r != ncclSuccess)
        return nccl_fail(r, "ncclGetVersion");
    *out = v;
    return 0;
}
