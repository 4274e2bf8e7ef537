// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" face over the UNMODIFIED reference headers under
// /root/reference/proj/include (compiled in place by oracle/Makefile into
// oracle/_ref/libsvdbref.so).  Nothing from the reference is copied here: every
// function below only calls reference entry points so that the Python tests,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// can drive the reference CPU implementation through ctypes.
//
// Reference entry points used (file:line under /root/reference/proj/include/svdb):
//   compress()            compress.hpp:221      serialize_frozen()  io.hpp:175
//   parse_frozen()        io.hpp:183            FrozenGrid::read_voxel frozen.hpp:82
//   Accessor::read        frozen.hpp:234        sample_field()      sample.hpp:74 (line 401 in cat)
//   build_macrocells()    macrocell.hpp:74      update_majorants()  macrocell.hpp:108
//   dda_traverse()        dda.hpp:52            woodcock_track()    render.hpp:106
//   render_field()        render.hpp:276        trace_path()        render.hpp:160
//   detail::camera_ray()  render.hpp:259        Rng::for_pixel_sample rng.hpp:45
//   SparseGridBuilder     tree.hpp:166 (set_voxel/set_tile/prune)   freeze() frozen.hpp:136

#include <svdb/svdb.hpp>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

using namespace svdb;

namespace {

thread_local std::string g_last_error;

int code_of(const Error& e) { return int(e.code()) + 1; }

template <typename F>
int guarded(F&& f)
{
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_last_error = e.what();
        return code_of(e);
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return 100;
    }
}

uint8_t* copy_out(const std::vector<std::uint8_t>& v, size_t* n)
{
    auto* p = static_cast<uint8_t*>(std::malloc(v.size() ? v.size() : 1));
    if (!v.empty())
        std::memcpy(p, v.data(), v.size());
    *n = v.size();
    return p;
}

struct RefGrid {
    FrozenGrid grid;
    std::unique_ptr<MacrocellGrid> mc;
};

TransferFunction make_tf(double lo, double hi, const float* rgba, int n, double scale)
{
    std::vector<std::array<float, 4>> e(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i)
        e[size_t(i)] = {rgba[4 * i], rgba[4 * i + 1], rgba[4 * i + 2], rgba[4 * i + 3]};
    return TransferFunction(lo, hi, std::move(e), scale);
}

Camera make_cam(const double* cam9, double fov, int w, int h)
{
    Camera c;
    c.position = {cam9[0], cam9[1], cam9[2]};
    c.look_at = {cam9[3], cam9[4], cam9[5]};
    c.up = {cam9[6], cam9[7], cam9[8]};
    c.fov_y_deg = fov;
    c.width = w;
    c.height = h;
    return c;
}

RenderSettings make_rs(int spp, int max_bounces, int rr_start, uint64_t seed, int mode, double iso,
                       const float* ambient, const float* bgcol, int threads)
{
    RenderSettings rs;
    rs.spp = spp;
    rs.max_bounces = max_bounces;
    rs.rr_start_bounce = rr_start;
    rs.seed = seed;
    rs.mode = mode == 1 ? RenderMode::iso : RenderMode::pathtrace;
    rs.iso_value = iso;
    rs.ambient_radiance = {ambient[0], ambient[1], ambient[2]};
    rs.background_color = {bgcol[0], bgcol[1], bgcol[2]};
    rs.threads = threads;
    return rs;
}

/// Field wrapper counting lattice reads (the reference's Field concept,
/// render.hpp:85-93); one counter per copy, summed by the caller.
struct CountingField {
    GridField inner;
    mutable std::uint64_t* counter;
    explicit CountingField(const FrozenGrid& g, std::uint64_t* c) : inner(g), counter(c) {}
    CountingField(const CountingField& o) : inner(o.inner), counter(o.counter) {}
    float operator()(const Coord& c) const
    {
        ++*counter;
        return inner(c);
    }
};

} // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }
void ref_free(void* p) { std::free(p); }

/// compress() a dense f32 volume (x fastest). voxel_type 0 = u8 source
/// (values must already be byte/255.0f as load_raw makes them), 1 = f32.
int ref_compress(const float* data, int dx, int dy, int dz, int voxel_type, double quality,
                 int metric, uint8_t** out, size_t* n_out, uint64_t* report7)
{
    return guarded([&] {
        std::vector<float> v(data, data + size_t(dx) * size_t(dy) * size_t(dz));
        DenseVolume vol = DenseVolume::from_data({dx, dy, dz}, std::move(v),
                                                 voxel_type == 0 ? VoxelType::u8 : VoxelType::f32);
        CompressionParams p;
        p.quality = quality;
        p.metric = Metric(metric);
        auto [g, rep] = compress(vol, p);
        *out = copy_out(serialize_frozen(g), n_out);
        if (report7) {
            std::memcpy(&report7[0], &rep.background, 4);
            report7[1] = rep.num_bricks;
            report7[2] = rep.bricks_activated;
            report7[3] = rep.voxels_activated;
            report7[4] = rep.frozen_bytes;
            report7[5] = rep.dense_bytes;
            std::memcpy(&report7[6], &rep.achieved_ratio, 8);
        }
    });
}

/// Builder op list -> frozen SVDB bytes. kind 0 = set_voxel, 1 = lower-slot
/// tile, 2 = upper-slot tile (tree.hpp:184-281). do_prune calls prune().
int ref_build_ops(int dx, int dy, int dz, float background, const int* kinds, const int* xyz,
                  const float* vals, size_t n_ops, int do_prune, uint8_t** out, size_t* n_out)
{
    return guarded([&] {
        SparseGridBuilder b({dx, dy, dz}, background);
        for (size_t i = 0; i < n_ops; ++i) {
            Coord c{xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
            if (kinds[i] == 0)
                b.set_voxel(c, vals[i]);
            else
                b.set_tile(kinds[i] == 1 ? TileLevel::lower_slot : TileLevel::upper_slot, c, vals[i]);
        }
        if (do_prune)
            b.prune();
        *out = copy_out(serialize_frozen(freeze(b)), n_out);
    });
}

int ref_grid_open(const uint8_t* bytes, size_t n, void** handle)
{
    return guarded([&] {
        auto* g = new RefGrid{parse_frozen(bytes, n), nullptr};
        *handle = g;
    });
}

void ref_grid_close(void* h) { delete static_cast<RefGrid*>(h); }

int ref_read_voxels(void* h, const int32_t* ijk, size_t n, float* out, int cached)
{
    return guarded([&] {
        const FrozenGrid& g = static_cast<RefGrid*>(h)->grid;
        Accessor acc(g);
        for (size_t i = 0; i < n; ++i) {
            Coord c{ijk[3 * i], ijk[3 * i + 1], ijk[3 * i + 2]};
            out[i] = cached ? acc.read(c) : g.read_voxel(c);
        }
    });
}

int ref_sample(void* h, const double* xyz, size_t n, int mode, float* out)
{
    return guarded([&] {
        Accessor acc(static_cast<RefGrid*>(h)->grid);
        for (size_t i = 0; i < n; ++i)
            out[i] = sample(acc, {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]},
                            mode == 0 ? SampleMode::nearest : SampleMode::trilinear);
    });
}

int ref_gradient(void* h, const double* xyz, size_t n, double* out)
{
    return guarded([&] {
        Accessor acc(static_cast<RefGrid*>(h)->grid);
        for (size_t i = 0; i < n; ++i) {
            Vec3d g = gradient(acc, {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]});
            out[3 * i] = g.x;
            out[3 * i + 1] = g.y;
            out[3 * i + 2] = g.z;
        }
    });
}

/// build_macrocells + update_majorants; arrays sized cell_count. cells3 out.
int ref_macrocells(void* h, double tf_lo, double tf_hi, const float* rgba, int n_entries,
                   double scale, int* cells3, float* cmin, float* cmax, float* maj, uint8_t* empty,
                   size_t cap, double* build_seconds)
{
    return guarded([&] {
        auto* rg = static_cast<RefGrid*>(h);
        auto t0 = std::chrono::steady_clock::now();
        MacrocellGrid mc = build_macrocells(rg->grid);
        TransferFunction tf = make_tf(tf_lo, tf_hi, rgba, n_entries, scale);
        update_majorants(mc, tf);
        auto t1 = std::chrono::steady_clock::now();
        if (build_seconds)
            *build_seconds = std::chrono::duration<double>(t1 - t0).count();
        cells3[0] = mc.cells.x;
        cells3[1] = mc.cells.y;
        cells3[2] = mc.cells.z;
        size_t nc = mc.cell_count();
        if (cmin && nc <= cap) {
            std::memcpy(cmin, mc.cell_min.data(), nc * 4);
            std::memcpy(cmax, mc.cell_max.data(), nc * 4);
            std::memcpy(maj, mc.majorant.data(), nc * 4);
            std::memcpy(empty, mc.empty.data(), nc);
        }
        rg->mc = std::make_unique<MacrocellGrid>(std::move(mc));
    });
}

/// dda_traverse KAT helper: writes up to cap visits (cell xyz, ta, tb).
int ref_dda(void* h, const double* ray6, double t0, double t1, int* cells, double* ts, size_t cap,
            size_t* n_visits)
{
    return guarded([&] {
        auto* rg = static_cast<RefGrid*>(h);
        MacrocellGrid mc = rg->mc ? *rg->mc : build_macrocells(rg->grid);
        Ray r{{ray6[0], ray6[1], ray6[2]}, {ray6[3], ray6[4], ray6[5]}};
        size_t k = 0;
        dda_traverse(mc, r, t0, t1, [&](const Vec3i& c, double ta, double tb) {
            if (k < cap) {
                cells[3 * k] = c.x;
                cells[3 * k + 1] = c.y;
                cells[3 * k + 2] = c.z;
                ts[2 * k] = ta;
                ts[2 * k + 1] = tb;
            }
            ++k;
            return true;
        });
        *n_visits = k;
    });
}

/// Full-frame svdb::render() (render.hpp:319): macrocells + majorants +
/// render_field(GridField). rgb = W*H*3 floats, row-major from the top row.
int ref_render(void* h, double tf_lo, double tf_hi, const float* rgba, int n_entries, double scale,
               const double* cam9, double fov, int w, int hgt, int spp, int max_bounces,
               int rr_start, uint64_t seed, int mode, double iso, const float* ambient,
               const float* bgcol, int threads, float* rgb)
{
    return guarded([&] {
        auto* rg = static_cast<RefGrid*>(h);
        TransferFunction tf = make_tf(tf_lo, tf_hi, rgba, n_entries, scale);
        Image img = render(rg->grid, tf, make_cam(cam9, fov, w, hgt),
                           make_rs(spp, max_bounces, rr_start, seed, mode, iso, ambient, bgcol,
                                   threads));
        std::memcpy(rgb, img.pixels.data(), img.pixels.size() * 12);
    });
}

} // extern "C"

/// Tile-subset render with the reference's per-pixel body (render.hpp:295-310) over macrocells
/// cached by ref_macrocells: only 16x16 tiles t with t % tile_stride == tile_phase are traced
/// (bounded CPU baseline samples). Pixels outside the subset are left untouched. With count != 0
/// every Field read goes through CountingField (8 per trilinear sample) and lookups_out gets the
/// total; with count == 0 the stock GridField (render.hpp:85-93) is used and lookups_out is 0, so a
/// timed baseline carries no instrumentation. threads = 0 uses all cores.
namespace {
template <typename MakeField>
void render_tile_subset(RefGrid* rg, const TransferFunction& tf, const Camera& cam, const RenderSettings& rs,
                        int w, int hgt, int spp, uint64_t seed, int threads, int tile_stride, int tile_phase,
                        float* rgb, uint64_t* paths_out, double* seconds, MakeField make_field)
{
    const MacrocellGrid& mc = *rg->mc;
    constexpr int tile = 16;
    int tiles_x = (w + tile - 1) / tile, tiles_y = (hgt + tile - 1) / tile;
    std::vector<int64_t> subset;
    for (int64_t t = 0; t < int64_t(tiles_x) * tiles_y; ++t)
        if (t % tile_stride == tile_phase)
            subset.push_back(t);
    std::atomic<uint64_t> paths{0};
    auto t0 = std::chrono::steady_clock::now();
    parallel_for(
        int64_t(subset.size()),
        [&](int64_t k) {
            auto local = make_field(k); // fresh Field (and Accessor) per tile, like render.hpp:292
            int64_t t = subset[size_t(k)];
            int tx = int(t % tiles_x) * tile, ty = int(t / tiles_x) * tile;
            uint64_t np = 0;
            for (int y = ty; y < std::min(ty + tile, hgt); ++y)
                for (int x = tx; x < std::min(tx + tile, w); ++x) {
                    Vec3d accum{0, 0, 0};
                    for (int s = 0; s < spp; ++s) {
                        Rng rng = Rng::for_pixel_sample(seed, x, y, s);
                        double jx = rng.uniform();
                        double jy = rng.uniform();
                        Ray ray = detail::camera_ray(cam, x + jx, y + jy);
                        Vec3f c = trace_path(local, mc, tf, ray, rs, rng);
                        accum += Vec3d{double(c.x), double(c.y), double(c.z)};
                        ++np;
                    }
                    accum /= double(spp);
                    size_t o = (size_t(y) * size_t(w) + size_t(x)) * 3;
                    rgb[o] = float(accum.x);
                    rgb[o + 1] = float(accum.y);
                    rgb[o + 2] = float(accum.z);
                }
            paths += np;
        },
        threads);
    auto t1 = std::chrono::steady_clock::now();
    *paths_out = paths.load();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
}
} // namespace

extern "C" {
int ref_render_tiles(void* h, double tf_lo, double tf_hi, const float* rgba, int n_entries,
                     double scale, const double* cam9, double fov, int w, int hgt, int spp,
                     int max_bounces, int rr_start, uint64_t seed, const float* ambient,
                     int threads, int tile_stride, int tile_phase, float* rgb,
                     uint64_t* lookups_out, uint64_t* paths_out, double* seconds, int count)
{
    return guarded([&] {
        auto* rg = static_cast<RefGrid*>(h);
        if (!rg->mc)
            fail(Errc::size_mismatch, "call ref_macrocells first");
        TransferFunction tf = make_tf(tf_lo, tf_hi, rgba, n_entries, scale);
        Camera cam = make_cam(cam9, fov, w, hgt);
        float bg[3] = {0, 0, 0};
        RenderSettings rs = make_rs(spp, max_bounces, rr_start, seed, 0, 0.5, ambient, bg, threads);
        *lookups_out = 0;
        if (count) {
            int tiles_x = (w + 15) / 16, tiles_y = (hgt + 15) / 16;
            std::vector<std::uint64_t> counts(size_t(tiles_x) * size_t(tiles_y), 0);
            render_tile_subset(rg, tf, cam, rs, w, hgt, spp, seed, threads, tile_stride, tile_phase, rgb, paths_out,
                               seconds, [&](int64_t k) { return CountingField(rg->grid, &counts[size_t(k)]); });
            for (auto c : counts)
                *lookups_out += c;
        } else {
            render_tile_subset(rg, tf, cam, rs, w, hgt, spp, seed, threads, tile_stride, tile_phase, rgb, paths_out,
                               seconds, [&](int64_t) { return GridField(rg->grid); });
        }
    });
}

/// Woodcock KAT helper (render.hpp:106-124): n independent trackings along
/// one ray with one Rng(seed) stream; t_out = event t or -1.
int ref_woodcock(void* h, double tf_lo, double tf_hi, const float* rgba, int n_entries,
                 double scale, double sigma_maj, const double* ray6, double t0, double t1,
                 uint64_t seed, size_t n, double* t_out, uint64_t* next_u64_after)
{
    return guarded([&] {
        auto* rg = static_cast<RefGrid*>(h);
        TransferFunction tf = make_tf(tf_lo, tf_hi, rgba, n_entries, scale);
        GridField field(rg->grid);
        Ray r{{ray6[0], ray6[1], ray6[2]}, {ray6[3], ray6[4], ray6[5]}};
        Rng rng(seed);
        for (size_t i = 0; i < n; ++i) {
            auto ev = woodcock_track(field, tf, sigma_maj, r, t0, t1, rng);
            t_out[i] = ev ? ev->t : -1.0;
        }
        if (next_u64_after)
            *next_u64_after = rng.next_u64();
    });
}

/// Rng stream KAT: n uniforms of for_pixel_sample(seed, px, py, s).
void ref_rng_uniforms(uint64_t seed, int px, int py, int s, size_t n, double* out)
{
    Rng rng = Rng::for_pixel_sample(seed, px, py, s);
    for (size_t i = 0; i < n; ++i)
        out[i] = rng.uniform();
}

int ref_hardware_threads() { return int(std::thread::hardware_concurrency()); }

} // extern "C"
