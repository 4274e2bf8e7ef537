// svdb_gpu_interop.hpp — drop-in overloads taking the reference's own types.
//
// Include AFTER the reference headers (<svdb/svdb.hpp>). A caller that today writes
//
//     svdb::Image img = svdb::render(grid, tf, cam, settings);          // render.hpp:319
//
// switches to the B200 path by writing
//
//     svdb::Image img = svdb::gpu::render(grid, tf, cam, settings);
//
// with the same argument types, the same Image layout (linear light, row 0 at the top) and the
// same exception type (svdb::Error carrying svdb::Errc; device failures surface as
// svdb::Error(Errc::io_error, "...") with the ABI message). The grid travels as the reference's
// own SVDB bytes (serialize_frozen, io.hpp:175) and is cached per FrozenGrid address by
// GridCache for repeated frames.
#pragma once

#include <map>
#include <mutex>

#include "svdb_gpu.hpp"

namespace svdb {
namespace gpu {

inline void rethrow_as_svdb(const Error& e)
{
    if (e.is_errc())
        throw svdb::Error(svdb::Errc(int(e.code())), e.what());
    throw svdb::Error(svdb::Errc::io_error, e.what());
}

inline TransferFunction convert(const svdb::TransferFunction& tf)
{
    TransferFunction t;
    t.domain_lo = tf.domain_lo();
    t.domain_hi = tf.domain_hi();
    t.density_scale = tf.density_scale();
    t.entries = tf.entries();
    return t;
}

inline Camera convert(const svdb::Camera& c)
{
    Camera o;
    o.position = {c.position.x, c.position.y, c.position.z};
    o.look_at = {c.look_at.x, c.look_at.y, c.look_at.z};
    o.up = {c.up.x, c.up.y, c.up.z};
    o.fov_y_deg = c.fov_y_deg;
    o.width = c.width;
    o.height = c.height;
    return o;
}

inline RenderSettings convert(const svdb::RenderSettings& s)
{
    RenderSettings o;
    o.spp = s.spp;
    o.max_bounces = s.max_bounces;
    o.rr_start_bounce = s.rr_start_bounce;
    o.seed = s.seed;
    o.mode = s.mode == svdb::RenderMode::iso ? RenderMode::iso : RenderMode::pathtrace;
    o.iso_value = s.iso_value;
    o.ambient_radiance = {s.ambient_radiance.x, s.ambient_radiance.y, s.ambient_radiance.z};
    o.background_color = {s.background_color.x, s.background_color.y, s.background_color.z};
    o.threads = s.threads;
    return o;
}

/// Upload a reference FrozenGrid (through its own serializer) to the GPU.
inline Grid upload(const svdb::FrozenGrid& g, Codec codec = Codec::f32, int device = 0)
{
    try {
        return Grid(svdb::serialize_frozen(g), codec, device);
    } catch (const Error& e) {
        rethrow_as_svdb(e);
    }
    throw svdb::Error(svdb::Errc::io_error, "unreachable");
}

/// Per-process cache: one device grid per FrozenGrid (frames re-render the same grid). Entries are
/// keyed by address and codec and validated by a fingerprint of the grid's shape and storage
/// (dims, background, node counts, vector data pointers, first/last leaf values), so a different
/// grid later constructed at the same address is re-uploaded instead of served stale. FrozenGrid
/// is immutable by contract (frozen.hpp:225-227); in-place edits of leaf values are not detected.
class GridCache {
public:
    static Grid& get(const svdb::FrozenGrid& g, Codec codec)
    {
        struct Entry {
            std::vector<uint64_t> fp;
            std::unique_ptr<Grid> grid;
        };
        static std::mutex mu;
        static std::map<std::pair<const svdb::FrozenGrid*, int>, Entry> cache;
        std::lock_guard<std::mutex> lk(mu);
        std::vector<uint64_t> fp = fingerprint(g);
        auto key = std::make_pair(&g, int(codec));
        auto it = cache.find(key);
        if (it != cache.end() && it->second.fp != fp) {
            cache.erase(it);
            it = cache.end();
        }
        if (it == cache.end())
            it = cache.emplace(key, Entry{fp, std::make_unique<Grid>(upload(g, codec))}).first;
        return *it->second.grid;
    }

private:
    static std::vector<uint64_t> fingerprint(const svdb::FrozenGrid& g)
    {
        auto bits = [](float f) {
            uint32_t u;
            std::memcpy(&u, &f, 4);
            return uint64_t(u);
        };
        std::vector<uint64_t> fp = {uint64_t(uint32_t(g.dims.x)), uint64_t(uint32_t(g.dims.y)),
                                    uint64_t(uint32_t(g.dims.z)), bits(g.background),
                                    g.root.size(), g.uppers.size(), g.lowers.size(), g.leaves.size(),
                                    uint64_t(reinterpret_cast<uintptr_t>(g.uppers.data())),
                                    uint64_t(reinterpret_cast<uintptr_t>(g.lowers.data())),
                                    uint64_t(reinterpret_cast<uintptr_t>(g.leaves.data()))};
        if (!g.leaves.empty()) {
            fp.push_back(bits(g.leaves.front().values.front()));
            fp.push_back(bits(g.leaves.back().values.back()));
        }
        return fp;
    }
};

/// Drop-in for svdb::render (render.hpp:319-325). codec F32 keeps the reference's values exactly.
inline svdb::Image render(const svdb::FrozenGrid& grid, const svdb::TransferFunction& tf, const svdb::Camera& cam,
                          const svdb::RenderSettings& settings, Codec codec = Codec::f32)
{
    try {
        Grid& g = GridCache::get(grid, codec);
        Image img = render(g, convert(tf), convert(cam), convert(settings));
        svdb::Image out;
        out.width = img.width;
        out.height = img.height;
        out.pixels.resize(img.pixels.size());
        for (size_t i = 0; i < img.pixels.size(); ++i)
            out.pixels[i] = svdb::Vec3f{img.pixels[i][0], img.pixels[i][1], img.pixels[i][2]};
        return out;
    } catch (const Error& e) {
        rethrow_as_svdb(e);
    }
    throw svdb::Error(svdb::Errc::io_error, "unreachable");
}

/// Drop-in for svdb::sample(const Accessor&, p, mode) (sample.hpp:97) over a device grid.
inline float sample(const svdb::FrozenGrid& grid, const svdb::Vec3d& p, svdb::SampleMode mode)
{
    try {
        Grid& g = GridCache::get(grid, Codec::f32);
        return sample(g, Vec3d{p.x, p.y, p.z}, mode == svdb::SampleMode::nearest ? SampleMode::nearest
                                                                                 : SampleMode::trilinear);
    } catch (const Error& e) {
        rethrow_as_svdb(e);
    }
    return 0.0f;
}

} // namespace gpu
} // namespace svdb
