// svdbgpu_internal.hpp — host-side internals shared by the C-ABI, the encoder and the kernels.
#pragma once

#include <cstdint>
#include <functional>
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

int compress(const float* data, const int32_t dims[3], int voxel_type, double quality, int metric,
             int threads, std::vector<uint8_t>& out, svdbgpu_compress_report* rep);
int synth(int kind, const int32_t dims[3], uint64_t seed, int threads, float* out);

} // namespace svdbgpu
