// svdbgpu_internal.hpp — host-side internals shared by the C-ABI, the encoder and the kernels.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <functional>
#include <new>
#include <string>
#include <vector>

#include "svdbgpu.h"

namespace svdbgpu {

// svdb::Errc (errors.hpp:11-23); the ABI returns value + 1.
enum class Errc {
    io_error,
    size_mismatch,
    non_finite_voxel,
    out_of_bounds,
    misaligned,
    empty_box,
    invalid_quality,
    bad_magic,
    version_mismatch,
    corrupt_index,
    dims_mismatch,
};

void set_error(const std::string& msg);
int fail(Errc code, const std::string& msg);  // records msg, returns int(code) + 1
int fail_code(int code, const std::string& msg);

int resolve_threads(int threads);
void parallel_for(int64_t n, int threads, const std::function<void(int64_t, int64_t, int)>& body);

// malloc'd, zero-filled output buffer handed to the caller of the C-ABI (freed with svdbgpu_free)
struct HostBuf {
    uint8_t* p = nullptr;
    size_t n = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() { std::free(p); }
    void alloc(size_t bytes)
    {
        std::free(p);
        p = static_cast<uint8_t*>(std::calloc(bytes ? bytes : 1, 1));
        if (!p)
            throw std::bad_alloc();
        n = bytes;
    }
    uint8_t* release()
    {
        uint8_t* q = p;
        p = nullptr;
        return q;
    }
};

int compress(const float* data, const int32_t dims[3], int voxel_type, double quality, int metric,
             int threads, HostBuf& out, svdbgpu_compress_report* rep);
int synth(int kind, const int32_t dims[3], uint64_t seed, int threads, float* out);
double sparse_threshold(int dim_max);
// the value-noise octaves of synth() (lattice of (cells+2)^3 values, scale = lattice units per voxel)
struct SynthOctave {
    int cells, n;
    double scale;
    std::vector<float> lat;
};
void synth_lattices(int kind, const int32_t dims[3], uint64_t seed, std::vector<SynthOctave>& out);
// streaming device encoder (stream_encoder.cu): z-slabs produced on the device or by a host callback
typedef int (*SlabFn)(void* user, int32_t z0, int32_t nz, float* out);
int stream_compress_synth(int kind, const int32_t dims[3], uint64_t seed, double quality, int metric, int device,
                          HostBuf& out, svdbgpu_compress_report* rep, double* seconds);
int stream_compress_callback(SlabFn fn, void* user, const int32_t dims[3], int voxel_type, double quality,
                             int metric, int device, HostBuf& out, svdbgpu_compress_report* rep, double* seconds);

// Encoder stages shared by the dense compress() and the streaming device encoder (stream_encoder.cu).
constexpr int kEncBrick = 32; // compress.hpp brick edge
enum : uint8_t { kBlkAbsent = 0, kBlkLeaf = 1, kBlkTile = 2, kBlkCornerLeaf = 3 }; // per 8^3 leaf block
void choose_bricks(const int32_t dims[3], const float* blo, const float* bhi, float bg, int metric, double quality,
                   std::vector<uint8_t>& chosen, uint64_t& budget, uint64_t& voxels_activated);
void write_tree(const int32_t dims[3], int voxel_type, float bg, float vmin, float vmax,
                const std::vector<uint8_t>& state, const std::vector<float>& tile_val, int threads,
                HostBuf& out, std::vector<uint32_t>& leaf_index, uint64_t& n_leaf, uint64_t& leaf_offset);

} // namespace svdbgpu
