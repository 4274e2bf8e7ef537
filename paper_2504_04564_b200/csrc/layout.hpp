// layout.hpp — plain device-layout structs shared by host (C++) and device (CUDA) code.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace svdbgpu {

// Bounds-checked debug build (-DSVDB_CHECKED=1, csrc/Makefile `variants`): device asserts on every
// indexed load / store of the hot path (tools/checked_run.sh). compute-sanitizer is closed on the
// GPU pool, so this is the memory-safety check of record.
#ifndef SVDB_CHECKED
#define SVDB_CHECKED 0
#endif
#if SVDB_CHECKED && defined(__CUDA_ARCH__)
#define SVDB_ASSERT(cond)                                                                      \
    do {                                                                                       \
        if (!(cond)) {                                                                         \
            printf("SVDB_ASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #cond);              \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define SVDB_ASSERT(cond) ((void)0)
#endif

enum SlotKind : uint32_t { kSlotBackground = 0, kSlotTile = 1, kSlotChild = 2 };

// Device tree. Node tables are pre-resolved at upload so one load answers "what is in this
// slot" with the reference's precedence (tile bit before child bit, frozen.hpp:88-97):
//   upper: uint2 {kind, payload}         payload = lower index | f32 tile bits
//   lower: uint4 {kind, payload, lo, sc} payload = leaf index | f32 tile bits; lo/sc = the
//          child leaf's decode parameters, so a leaf miss costs one 16-B load + the codes.
// Leaf payloads are one contiguous array, leaf i at codes + i * leaf_stride.
struct DevGrid {
    int dims[3];
    float background;
    int n_root;
    const int4* root; // {origin x, y, z, upper index}, file order (z,y,x sorted)
    const uint2* upper;
    const uint4* lower;
    const uint8_t* codes;
    float2* lparams;      // 8 x (lo, scale) per leaf: [0] own, [1..7] apron regions
    uint32_t leaf_stride; // bytes per leaf: the 9^3 stencil brick (own 8^3 block + 217-voxel apron)
    uint32_t main_bytes;  // the own block in the reference's voxel order (v2 container): 2048 f32, 512 u8, 256 u4
    uint32_t n_leaf, n_lower;
    // leaf directory: for every 8^3 block of [0, 8*dir_dims) the root->upper->lower walk resolved
    // at build time ({kind, payload, lo, scale} as in `lower`; tile / background as kind tile with
    // the value). One load replaces the node walk for in-box lookups; null when over budget.
    const uint4* dir;
    int dir_dims[3];
};

struct DevTF {
    double lo, hi, scale;
    int n;
    // 1 / (hi - lo) when hi - lo is a power of two (then (v - lo) * inv_range == (v - lo) / (hi - lo)
    // exactly and the per-lookup FP64 division is skipped), else 0
    double inv_range;
};

// Transfer-function entries are staged in shared memory up to this many (16 KB); larger tables are
// read from global memory (L1-cached) so any entry count the reference accepts renders.
constexpr int kTfSmemMax = 1024;
__host__ __device__ inline size_t tf_smem_bytes(int n) { return n <= kTfSmemMax ? size_t(n) * 16 : 0; }

constexpr int kCodecF32 = 0, kCodecUnorm8 = 1, kCodecAffine8 = 2, kCodecAffine4 = 3;

} // namespace svdbgpu
