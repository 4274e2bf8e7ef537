// render_args.hpp — launch arguments shared by the FP64 reference-exact kernels (render.cu) and
// the FP32 tracking kernel (render_fast.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "layout.hpp"

namespace svdbgpu {

struct CamArgs {
    double pos[3], fwd[3], right[3], up[3];
    double tan_half, aspect;
    int w, h;
};

struct RenderArgs {
    DevGrid g;
    DevTF tf;
    const float4* tf_ent;
    const float* maj;
    const double* inv_maj;
    const float* inv_maj_f; // float(1 / majorant), 0 for cells without draws (FP32 tracking)
    const float* cmin;
    const float* cmax;
    // hierarchical DDA (settings.hdda): 128^3 lower-node regions over the majorant grid; cdraw[c] != 0
    // when some majorant cell inside region c has draws
    int ccells[3];
    const uint8_t* cdraw;
    int cells[3];
    double cell;  // majorant cell edge in voxels (32 = the reference's MacrocellGrid::cell_dim)
    double icell; // 1/cell, exact (cell is a power of two), so e * icell == e / cell bit for bit
    double hi[3];
    CamArgs cam;
    int spp, max_bounces, rr_start;
    uint64_t seed_mixed;
    double iso;
    float ambient[3], background[3];
    double ea_step, ea_min_t;
    int rank, nranks, tiles_x;
    float* out;
    int packed;
    unsigned long long* counters;
    // sample-chunked work (chunk > 0): a work item is (8x4 pixel block, `chunk` consecutive samples);
    // each sample's float RGB goes to sbuf[(pixel * spp + s) * 3] and k_reduce sums a pixel's
    // samples in index order in FP64 afterwards (render.hpp:297-310). chunk == 0: a lane owns a
    // whole pixel and accumulates in place.
    float* sbuf;
    int chunk, nchunks;
    // sample-chunked renders: camera rays precomputed at full SIMD width by k_camera_rays, per
    // (pixel, sample) as sbuf: {d.x, d.y}, {d.z, RNG state after the two jitter draws} (32 B)
    const double2* camtab;
    long long npix; // pixel slots of out / sbuf / camtab (packed: this rank's tiles x 256)
};

// FP32-arithmetic tracking kernel launch (render_fast.cu): SVDBGPU_PRECISION_FP32 (all FP32) or
// SVDBGPU_PRECISION_MIXED (FP64 ray / DDA / distances, FP32 for the rest); persistent grid sized
// from occupancy.
int launch_trace_fast(const RenderArgs& A, int codec, int mode, int precision, long long n_units, size_t smem,
                      cudaStream_t s);

} // namespace svdbgpu
