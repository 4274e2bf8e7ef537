// grid_impl.hpp — host-side state of one device-resident grid (behind svdbgpu_grid*).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "layout.hpp"
#include "svdbgpu.h"
#include "svdbgpu_internal.hpp"

namespace svdbgpu {

int cuda_fail(cudaError_t e, const char* what);

// NVTX range for the host phases (visible in nsys / ncu timelines; no-op without a tool attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

#define SVDB_CUDA(call)                                                                        \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            return ::svdbgpu::cuda_fail(e_, #call);                                            \
    } while (0)

struct GridImpl {
    int device = 0;
    int codec = 0;
    int voxel_type = 1;
    float value_domain[2] = {0, 0};
    uint64_t n_upper = 0, n_lower = 0, n_leaf = 0, n_root = 0, svdb_bytes = 0;
    DevGrid dg{};
    int4* d_root = nullptr;
    uint2* d_upper = nullptr;
    uint4* d_lower = nullptr;
    uint8_t* d_codes = nullptr;
    float2* d_lparams = nullptr;
    uint4* d_dir = nullptr; // leaf directory (DevGrid::dir)
    uint64_t device_bytes = 0, leaf_payload_bytes = 0;

    // macrocells: exact closed-box ranges cached per grid (macrocell.hpp:74-103);
    // majorants recomputed per TF (macrocell.hpp:108-116). cell_dim 32 is the reference's
    // (MacrocellGrid::cell_dim); 128 / 8 are the lower-node / leaf-node majorant grids of the
    // node-majorant tracking mode.
    int cell_dim = 32;
    int cells[3] = {0, 0, 0};
    float* d_cmin = nullptr;
    float* d_cmax = nullptr;
    float* d_maj = nullptr;
    double* d_inv_maj = nullptr; // 1.0 / double(majorant), 0 for empty cells
    float* d_inv_maj_f = nullptr; // the same in float (FP32 tracking kernel)
    bool ranges_valid = false;
    uint8_t* d_cdraw = nullptr; // hierarchical DDA: per 128^3 region, "some majorant cell has draws"
    size_t cdraw_cap = 0;
    float4* d_tf = nullptr;
    int tf_cap = 0;
    float* d_img = nullptr;
    float* d_gather = nullptr; // multi-device render: packed tiles of every device (first device only)
    size_t gather_cap = 0;
    float* d_sbuf = nullptr; // per-sample results of sample-chunked renders
    size_t sbuf_cap = 0;
    double2* d_camtab = nullptr; // precomputed camera rays of sample-chunked renders
    size_t camtab_cap = 0;
    size_t img_cap = 0;
    unsigned long long* d_counters = nullptr;
    double* d_scratch = nullptr;
    size_t scratch_cap = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::mutex mu;

    ~GridImpl();
    int ensure_ranges(cudaStream_t s, float* ms, int cell_dim = 32);
    int upload_tf(const svdbgpu_tf* tf, cudaStream_t s, DevTF* out);
};

int validate_tf(const svdbgpu_tf* tf);
int grid_create(const uint8_t* svdb, size_t n, int codec, int device, GridImpl** out);
int grid_leaf_codes(const GridImpl* g, uint64_t first, uint64_t count, uint8_t* codes, float* params);
int quantise_svdb(const uint8_t* svdb, size_t n, int codec, int device, std::vector<uint8_t>& out);
int read_voxels_device(const GridImpl* g, const int32_t* d_ijk, size_t n, float* d_out, cudaStream_t s);
int sample_device(const GridImpl* g, const double* d_xyz, size_t n, int mode, float* d_out, cudaStream_t s);
int gradient_device(const GridImpl* g, const double* d_xyz, size_t n, double* d_out, cudaStream_t s);
int majorants(GridImpl* g, const DevTF& tf, cudaStream_t s, uint8_t* d_empty = nullptr);
int coarse_flags(GridImpl* g, const int ccells[3], cudaStream_t s);
int render(GridImpl* g, const svdbgpu_tf* tf, const svdbgpu_camera* cam, const svdbgpu_settings* st,
           float* d_out, int packed, cudaStream_t s, svdbgpu_stats* stats);
int unpack_tiles(const float* d_packed, int nranks, int64_t max_tiles, int w, int h, float* d_rgb,
                 cudaStream_t s);
int64_t tiles_for_rank(int w, int h, int rank, int nranks);

} // namespace svdbgpu

// The opaque handle of the C-ABI (include/svdbgpu.h).
struct svdbgpu_grid {
    std::unique_ptr<svdbgpu::GridImpl> impl;
};
