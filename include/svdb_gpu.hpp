// svdb_gpu.hpp — header-only C++ mirror of the reference svdb hot-path API over the C-ABI
// (svdbgpu.h / libsvdbgpu.so). Same names, argument meaning and error behaviour as
// /root/reference/proj/include/svdb (exceptions carrying Errc, never status returns):
//
//   svdb::gpu::Grid              <- FrozenGrid (frozen.hpp:70-131), resident on one GPU
//   Grid::read_voxel             <- FrozenGrid::read_voxel (frozen.hpp:82-99)
//   svdb::gpu::sample / gradient <- sample / gradient (sample.hpp:97-105)
//   svdb::gpu::render            <- render (render.hpp:319-325)
//   svdb::gpu::compress          <- compress + serialize_frozen (compress.hpp:221, io.hpp:175)
//
// With the reference headers also included, svdb_gpu_interop.hpp adds overloads that take the
// reference's own types (svdb::FrozenGrid, svdb::TransferFunction, ...) and throw svdb::Error.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "svdbgpu.h"

namespace svdb {
namespace gpu {

enum class Errc { // errors.hpp:11-23
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

/// svdb::Error equivalent; status() is the raw ABI code (1..11 = Errc + 1, or SVDBGPU_E_*).
class Error : public std::runtime_error {
public:
    Error(int status, const std::string& what) : std::runtime_error(what), status_(status) {}
    int status() const { return status_; }
    bool is_errc() const { return status_ >= 1 && status_ <= 11; }
    Errc code() const { return Errc(is_errc() ? status_ - 1 : 0); }

private:
    int status_;
};

inline void check(int rc)
{
    if (rc != SVDBGPU_OK) {
        const char* m = svdbgpu_last_error();
        throw Error(rc, m ? m : "svdbgpu error");
    }
}

enum class Codec : int32_t { f32 = SVDBGPU_CODEC_F32, unorm8 = SVDBGPU_CODEC_UNORM8,
                             affine8 = SVDBGPU_CODEC_AFFINE8, affine4 = SVDBGPU_CODEC_AFFINE4,
                             auto8 = SVDBGPU_CODEC_AUTO8 };
enum class SampleMode { nearest, trilinear };
enum class RenderMode : int32_t { pathtrace = SVDBGPU_MODE_PATHTRACE, iso = SVDBGPU_MODE_ISO,
                                  ea = SVDBGPU_MODE_EA, ratio = SVDBGPU_MODE_RATIO };
enum class Metric : int32_t { closest, farthest, median };
enum class VoxelType : int32_t { u8 = 0, f32 = 1 };

using Coord = std::array<int32_t, 3>;
using Vec3d = std::array<double, 3>;
using Vec3f = std::array<float, 3>;

/// transfer.hpp:23-35 (validated by the library with the same Errc::size_mismatch cases)
struct TransferFunction {
    double domain_lo = 0.0, domain_hi = 1.0;
    std::vector<std::array<float, 4>> entries;
    double density_scale = 1.0;

    svdbgpu_tf c() const
    {
        return svdbgpu_tf{domain_lo, domain_hi, density_scale, int32_t(entries.size()),
                          entries.empty() ? nullptr : entries[0].data()};
    }
};

/// render.hpp:25-32
struct Camera {
    Vec3d position{0, 0, 0};
    Vec3d look_at{0, 0, 1};
    Vec3d up{0, 1, 0};
    double fov_y_deg = 45.0;
    int width = 512;
    int height = 512;

    svdbgpu_camera c() const
    {
        svdbgpu_camera r{};
        for (int a = 0; a < 3; ++a) {
            r.position[a] = position[size_t(a)];
            r.look_at[a] = look_at[size_t(a)];
            r.up[a] = up[size_t(a)];
        }
        r.fov_y_deg = fov_y_deg;
        r.width = width;
        r.height = height;
        return r;
    }
};

/// render.hpp:39-49 (+ EA step/threshold; `threads` accepted for signature parity and ignored)
struct RenderSettings {
    int spp = 16;
    int max_bounces = 64;
    int rr_start_bounce = 3;
    uint64_t seed = 0;
    RenderMode mode = RenderMode::pathtrace;
    double iso_value = 0.5;
    Vec3f ambient_radiance{1.0f, 1.0f, 1.0f};
    Vec3f background_color{0.0f, 0.0f, 0.0f};
    int threads = 0;
    double ea_step = 0.5;
    double ea_min_transmittance = 1e-4;
    int tile_rank = 0, tile_nranks = 1;
    int majorant_cell = 0; // 0/32 reference macrocells; 8 / 128 node-majorant grids
    int precision = 0;     // SVDBGPU_PRECISION_FP64 (bit parity) / SVDBGPU_PRECISION_FP32
    int hdda = 0;          // 1: hierarchical empty-space skipping over the node tree

    svdbgpu_settings c() const
    {
        svdbgpu_settings s{};
        s.spp = spp;
        s.max_bounces = max_bounces;
        s.rr_start_bounce = rr_start_bounce;
        s.seed = seed;
        s.mode = int32_t(mode);
        s.iso_value = iso_value;
        for (int a = 0; a < 3; ++a) {
            s.ambient[a] = ambient_radiance[size_t(a)];
            s.background[a] = background_color[size_t(a)];
        }
        s.ea_step = ea_step;
        s.ea_min_transmittance = ea_min_transmittance;
        s.tile_rank = tile_rank;
        s.tile_nranks = tile_nranks;
        s.majorant_cell = majorant_cell;
        s.precision = precision;
        s.hdda = hdda;
        return s;
    }
};

/// render.hpp:51-58: linear light, pixels[y * width + x], row 0 at the top
struct Image {
    int width = 0;
    int height = 0;
    std::vector<Vec3f> pixels;
    svdbgpu_stats stats{};
    const Vec3f& at(int x, int y) const { return pixels[size_t(y) * size_t(width) + size_t(x)]; }
};

/// A frozen grid resident on one GPU. Immutable; thread-safe for lookups and renders.
class Grid {
public:
    explicit Grid(const std::vector<uint8_t>& svdb, Codec codec = Codec::auto8, int device = 0)
        : Grid(svdb.data(), svdb.size(), codec, device)
    {
    }
    Grid(const uint8_t* svdb, size_t n, Codec codec = Codec::auto8, int device = 0)
    {
        svdbgpu_grid* g = nullptr;
        check(svdbgpu_grid_create(svdb, n, int32_t(codec), device, &g));
        h_.reset(g);
        check(svdbgpu_grid_info_get(g, &info_));
    }

    const svdbgpu_grid_info& info() const { return info_; }
    svdbgpu_grid* handle() const { return h_.get(); }
    float background() const { return info_.background; }

    float read_voxel(const Coord& ijk) const
    {
        float v = 0.0f;
        check(svdbgpu_read_voxels(h_.get(), ijk.data(), 1, &v));
        return v;
    }
    std::vector<float> read_voxels(const std::vector<Coord>& ijk) const
    {
        std::vector<float> out(ijk.size());
        if (!ijk.empty())
            check(svdbgpu_read_voxels(h_.get(), ijk[0].data(), ijk.size(), out.data()));
        return out;
    }

private:
    struct Del {
        void operator()(svdbgpu_grid* g) const { svdbgpu_grid_destroy(g); }
    };
    std::unique_ptr<svdbgpu_grid, Del> h_;
    svdbgpu_grid_info info_{};
};

inline float sample(const Grid& g, const Vec3d& p, SampleMode mode)
{
    float v = 0.0f;
    check(svdbgpu_sample(g.handle(), p.data(), 1, mode == SampleMode::nearest ? 0 : 1, &v));
    return v;
}

inline std::vector<float> sample(const Grid& g, const std::vector<Vec3d>& p, SampleMode mode)
{
    std::vector<float> out(p.size());
    if (!p.empty())
        check(svdbgpu_sample(g.handle(), p[0].data(), p.size(), mode == SampleMode::nearest ? 0 : 1, out.data()));
    return out;
}

inline Vec3d gradient(const Grid& g, const Vec3d& p)
{
    Vec3d out{};
    check(svdbgpu_gradient(g.handle(), p.data(), 1, out.data()));
    return out;
}

/// build_macrocells + update_majorants (macrocell.hpp:74-116)
struct Macrocells {
    std::array<int32_t, 3> cells{};
    std::vector<float> cell_min, cell_max, majorant;
    std::vector<uint8_t> empty;
};

inline Macrocells macrocells(Grid& g, const TransferFunction& tf)
{
    Macrocells m;
    svdbgpu_tf t = tf.c();
    check(svdbgpu_macrocells(g.handle(), &t, m.cells.data(), nullptr, nullptr, nullptr, nullptr, 0));
    size_t n = size_t(m.cells[0]) * size_t(m.cells[1]) * size_t(m.cells[2]);
    m.cell_min.resize(n);
    m.cell_max.resize(n);
    m.majorant.resize(n);
    m.empty.resize(n);
    check(svdbgpu_macrocells(g.handle(), &t, m.cells.data(), m.cell_min.data(), m.cell_max.data(),
                             m.majorant.data(), m.empty.data(), n));
    return m;
}

/// render(grid, tf, cam, settings) (render.hpp:319-325) on the GPU
inline Image render(Grid& g, const TransferFunction& tf, const Camera& cam, const RenderSettings& rs)
{
    Image img;
    img.width = cam.width;
    img.height = cam.height;
    img.pixels.assign(size_t(cam.width) * size_t(cam.height), Vec3f{0, 0, 0});
    svdbgpu_tf t = tf.c();
    svdbgpu_camera c = cam.c();
    svdbgpu_settings s = rs.c();
    check(svdbgpu_render(g.handle(), &t, &c, &s, img.pixels[0].data(), &img.stats));
    return img;
}

/// render() over several devices from one process: grids[k] holds the same SVDB on device k's id;
/// interleaved 16x16 tiles per device, one NCCL gather, the frame bit-identical to render()
/// (svdbgpu_render_multi). gather_ms (optional) receives the gather's device time.
inline Image render(const std::vector<Grid*>& grids, const TransferFunction& tf, const Camera& cam,
                    const RenderSettings& rs, double* gather_ms = nullptr)
{
    Image img;
    img.width = cam.width;
    img.height = cam.height;
    img.pixels.assign(size_t(cam.width) * size_t(cam.height), Vec3f{0, 0, 0});
    std::vector<svdbgpu_grid*> h;
    for (Grid* g : grids)
        h.push_back(g ? g->handle() : nullptr);
    svdbgpu_tf t = tf.c();
    svdbgpu_camera c = cam.c();
    svdbgpu_settings s = rs.c();
    check(svdbgpu_render_multi(h.data(), int32_t(h.size()), &t, &c, &s, img.pixels[0].data(), &img.stats, gather_ms));
    return img;
}

struct CompressionParams { // compress.hpp:68-76
    double quality = 1.0;
    Metric metric = Metric::median;
};

/// compress + serialize_frozen: SVDB v1 bytes of a dense x-fastest volume (byte-identical to
/// the reference's output; u8 sources must hold byte/255.0f values, volume.hpp:91-97)
inline std::vector<uint8_t> compress(const float* data, const std::array<int32_t, 3>& dims,
                                     VoxelType type = VoxelType::f32, const CompressionParams& p = {},
                                     svdbgpu_compress_report* report = nullptr, int threads = 0)
{
    uint8_t* out = nullptr;
    size_t n = 0;
    check(svdbgpu_compress(data, dims.data(), int32_t(type), p.quality, int32_t(p.metric), threads, &out, &n, report));
    std::vector<uint8_t> v(out, out + n);
    svdbgpu_free(out);
    return v;
}

/// SVDB v1 -> quantised SVDB v2 (N-bit leaf codes + per-leaf lo/scale, encoded by the device codec);
/// Grid(v2) equals Grid(v1, codec).
inline std::vector<uint8_t> quantise(const std::vector<uint8_t>& svdb, Codec codec = Codec::auto8, int device = 0)
{
    uint8_t* out = nullptr;
    size_t n = 0;
    check(svdbgpu_quantise(svdb.data(), svdb.size(), int32_t(codec), device, &out, &n));
    std::vector<uint8_t> v(out, out + n);
    svdbgpu_free(out);
    return v;
}

} // namespace gpu
} // namespace svdb
