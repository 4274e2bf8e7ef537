// tests/cpp/test_interop.cpp — TEST INFRASTRUCTURE: the C++ drop-in (include/svdb_gpu.hpp +
// svdb_gpu_interop.hpp) used exactly the way a reference caller would, checked against the
// UNMODIFIED reference (headers from /root/reference/proj/include, compiled in place by
// tests/cpp/Makefile). Prints one PASS/FAIL line per check like the reference's acceptance.cpp;
// exit code = number of failures. Needs a GPU to run (built anywhere).
#include <svdb/svdb.hpp>

#include "svdb_gpu_interop.hpp"

#include <cmath>
#include <cstdio>

namespace {

int failures = 0;

void report(const char* name, bool ok, const std::string& detail = "")
{
    std::printf("%s %s %s\n", ok ? "PASS" : "FAIL", name, detail.c_str());
    failures += ok ? 0 : 1;
}

} // namespace

int main()
{
    using namespace svdb;
    // the reference's own pipeline (demo/pipeline_demo.cpp:17-55 shape)
    DenseVolume volume = synth_blobs({72, 64, 56}, 42, 10);
    CompressionParams params;
    params.quality = 0.5;
    auto [grid, rep] = compress(volume, params);

    // 1. encoder: svdb::gpu::compress == serialize_frozen(compress(...).first)
    {
        std::vector<uint8_t> mine = gpu::compress(volume.data().data(), {72, 64, 56}, gpu::VoxelType::f32,
                                                  gpu::CompressionParams{0.5, gpu::Metric::median});
        report("encoder_bytes_identical", mine == serialize_frozen(grid));
    }

    TransferFunction tf(0.0, double(volume.max_value()),
                        {{{0.1f, 0.1f, 0.8f, 0.0f}}, {{0.2f, 0.8f, 0.8f, 0.25f}}, {{0.9f, 0.9f, 0.2f, 0.6f}},
                         {{0.9f, 0.3f, 0.1f, 0.9f}}},
                        0.5);
    Camera cam;
    cam.look_at = {35.5, 31.5, 27.5};
    cam.position = {95.0, 76.0, -120.0};
    cam.width = 96;
    cam.height = 80;
    RenderSettings rs;
    rs.spp = 8;
    rs.seed = 1;

    // 2. render drop-in: same signature, same Image
    {
        Image want = render(grid, tf, cam, rs);
        Image got = gpu::render(grid, tf, cam, rs);
        size_t same = 0;
        double num = 0.0, den = 0.0;
        for (size_t i = 0; i < want.pixels.size(); ++i) {
            const Vec3f &a = got.pixels[i], &b = want.pixels[i];
            same += (std::memcmp(&a, &b, sizeof a) == 0);
            for (int c = 0; c < 3; ++c) {
                num += (double(a[c]) - double(b[c])) * (double(a[c]) - double(b[c]));
                den += double(b[c]) * double(b[c]);
            }
        }
        double rmse = std::sqrt(num / std::max(den, 1e-300));
        char buf[128];
        std::snprintf(buf, sizeof buf, "identical %.4f rel_rmse %.2e", double(same) / double(want.pixels.size()), rmse);
        report("render_drop_in", got.width == want.width && got.height == want.height && rmse <= 1e-3, buf);
        rs.mode = RenderMode::iso;
        rs.iso_value = 0.4;
        rs.spp = 2;
        Image wi = render(grid, tf, cam, rs);
        Image gi = gpu::render(grid, tf, cam, rs);
        size_t si = 0;
        for (size_t i = 0; i < wi.pixels.size(); ++i)
            si += (std::memcmp(&wi.pixels[i], &gi.pixels[i], sizeof(Vec3f)) == 0);
        report("iso_drop_in", si >= wi.pixels.size() * 99 / 100);
        // multi-device drop-in (svdbgpu_render_multi) over the devices visible here: the same frame
        rs.mode = RenderMode::pathtrace;
        rs.spp = 4;
        int32_t ndev = 0;
        svdbgpu_device_count(&ndev);
        std::vector<int> devs;
        for (int d = 0; d < ndev && d < 8; ++d)
            devs.push_back(d);
        Image one = gpu::render(grid, tf, cam, rs);
        Image many = gpu::render(grid, tf, cam, rs, devs);
        bool eq = one.pixels.size() == many.pixels.size();
        for (size_t i = 0; eq && i < one.pixels.size(); ++i)
            eq = std::memcmp(&one.pixels[i], &many.pixels[i], sizeof(Vec3f)) == 0;
        char mb[48];
        std::snprintf(mb, sizeof mb, "%zu device(s)", devs.size());
        report("render_multi_device_drop_in", eq && !devs.empty(), mb);
    }

    // 3. sampler drop-in: bit-exact against sample(Accessor) (sample.hpp:97)
    {
        Accessor acc(grid);
        Rng rng(9);
        bool ok = true;
        for (int i = 0; i < 20000 && ok; ++i) {
            Vec3d p{rng.uniform() * 90 - 9, rng.uniform() * 80 - 8, rng.uniform() * 70 - 7};
            ok = sample(acc, p, SampleMode::trilinear) == gpu::sample(grid, p, SampleMode::trilinear);
        }
        report("sample_bit_exact", ok);
    }

    // 5. acceptance criterion 6 (acceptance.cpp:169-199) through the GPU sampler: a lossless grid
    //    sampled at 1e5 random positions equals a dense trilinear oracle within 1e-6
    {
        DenseVolume v = synth_blobs({64, 64, 64}, 31, 7);
        auto [g6, r6] = compress(v, CompressionParams{});
        gpu::Grid dg = gpu::upload(g6, gpu::Codec::f32);
        Rng rng(606);
        std::vector<gpu::Vec3d> pts(100000);
        for (auto& p : pts)
            p = {rng.uniform() * 80.0 - 8.0, rng.uniform() * 80.0 - 8.0, rng.uniform() * 80.0 - 8.0};
        std::vector<float> got = gpu::sample(dg, pts, gpu::SampleMode::trilinear);
        auto dense_read = [&](const Coord& p) -> double {
            return v.contains(p) ? double(v.at(p)) : double(g6.background);
        };
        double worst = 0.0;
        for (size_t i = 0; i < pts.size(); ++i) {
            const auto& p = pts[i];
            int x0 = int(std::floor(p[0])), y0 = int(std::floor(p[1])), z0 = int(std::floor(p[2]));
            double fx = p[0] - x0, fy = p[1] - y0, fz = p[2] - z0, want = 0.0;
            for (int dz = 0; dz < 2; ++dz)
                for (int dy = 0; dy < 2; ++dy)
                    for (int dx = 0; dx < 2; ++dx)
                        want += (dx ? fx : 1 - fx) * (dy ? fy : 1 - fy) * (dz ? fz : 1 - fz) *
                                dense_read({x0 + dx, y0 + dy, z0 + dz});
            worst = std::max(worst, std::abs(double(got[i]) - want));
        }
        char buf[64];
        std::snprintf(buf, sizeof buf, "worst %.2e", worst);
        report("acceptance6_sampler_oracle", worst <= 1e-6, buf);
    }

    // 6. acceptance criterion 12 (acceptance.cpp:483-529): repeat renders identical, and the GPU
    //    frame equals the reference's render_field with a dense-sampler substitution
    {
        DenseVolume v = synth_blobs({64, 64, 64}, 17, 7);
        auto [g12, r12] = compress(v, CompressionParams{});
        TransferFunction tf12(0.0, double(v.max_value()), {{{0.3f, 0.7f, 0.9f, 0.0f}}, {{0.9f, 0.5f, 0.2f, 0.85f}}},
                              3.0);
        MacrocellGrid mc = build_macrocells(g12);
        update_majorants(mc, tf12);
        Camera c12;
        c12.position = {20.0, 45.0, -110.0};
        c12.look_at = {31.5, 31.5, 31.5};
        c12.width = 128;
        c12.height = 128;
        RenderSettings r;
        r.spp = 16;
        r.seed = 4096;
        Image one = gpu::render(g12, tf12, c12, r);
        Image two = gpu::render(g12, tf12, c12, r);
        struct DenseReader {
            const DenseVolume* v;
            float background;
            float operator()(const Coord& p) const { return v->contains(p) ? v->at(p) : background; }
        };
        Image dense = render_field(DenseReader{&v, g12.background}, mc, tf12, c12, r);
        size_t rep_same = 0, dense_same = 0;
        for (size_t i = 0; i < one.pixels.size(); ++i) {
            rep_same += std::memcmp(&one.pixels[i], &two.pixels[i], sizeof(Vec3f)) == 0;
            dense_same += std::memcmp(&one.pixels[i], &dense.pixels[i], sizeof(Vec3f)) == 0;
        }
        char buf[96];
        std::snprintf(buf, sizeof buf, "repeat %zu/%zu dense %zu/%zu", rep_same, one.pixels.size(), dense_same,
                      one.pixels.size());
        report("acceptance12_determinism_dense_substitution",
               rep_same == one.pixels.size() && dense_same >= one.pixels.size() * 98 / 100, buf);
    }

    // 7. GridCache: a different grid at the same address is re-uploaded, not served stale
    {
        auto* slot = new FrozenGrid(compress(synth_blobs({32, 32, 32}, 5, 3), CompressionParams{}).first);
        float a = gpu::sample(*slot, Vec3d{16.25, 16.5, 16.75}, SampleMode::trilinear);
        *slot = compress(synth_blobs({40, 40, 40}, 6, 4), CompressionParams{}).first;
        float b = gpu::sample(*slot, Vec3d{16.25, 16.5, 16.75}, SampleMode::trilinear);
        Accessor acc(*slot);
        report("grid_cache_revalidates", b == sample(acc, Vec3d{16.25, 16.5, 16.75}, SampleMode::trilinear) && a != b);
        gpu::GridCache::evict(*slot);
        delete slot;
    }

    // 7b. GridCache is bounded (LRU by device bytes) and evictable; a held grid outlives eviction
    {
        gpu::GridCache::clear();
        FrozenGrid g1 = compress(synth_blobs({32, 32, 32}, 5, 3), CompressionParams{}).first;
        FrozenGrid g2 = compress(synth_blobs({40, 40, 40}, 6, 4), CompressionParams{}).first;
        std::shared_ptr<gpu::Grid> h1 = gpu::GridCache::get(g1, gpu::Codec::f32);
        const uint64_t one = gpu::GridCache::resident_bytes();
        const uint64_t old_budget = gpu::GridCache::budget();
        gpu::GridCache::set_budget(one); // room for one grid only
        std::shared_ptr<gpu::Grid> h2 = gpu::GridCache::get(g2, gpu::Codec::f32);
        const bool lru = gpu::GridCache::size() == 1;
        // h1 was evicted from the cache but is still usable through the shared handle
        float v = gpu::sample(*h1, gpu::Vec3d{16.25, 16.5, 16.75}, gpu::SampleMode::trilinear);
        Accessor acc1(g1);
        const bool alive = v == sample(acc1, Vec3d{16.25, 16.5, 16.75}, SampleMode::trilinear);
        gpu::GridCache::evict(g2);
        const bool evicted = gpu::GridCache::size() == 0 && gpu::GridCache::resident_bytes() == 0;
        gpu::GridCache::set_budget(old_budget);
        report("grid_cache_bounded_lru_evict", lru && alive && evicted);
    }

    // 4. error mapping: corrupt containers raise the reference's Errc
    {
        std::vector<uint8_t> bytes = serialize_frozen(grid);
        bytes[0] = 'X';
        bool ok = false;
        try {
            gpu::Grid g(bytes);
        } catch (const gpu::Error& e) {
            ok = e.is_errc() && e.code() == gpu::Errc::bad_magic;
        }
        report("bad_magic_errc", ok);
        bytes[0] = 'S';
        bytes.pop_back();
        ok = false;
        try {
            gpu::Grid g(bytes);
        } catch (const gpu::Error& e) {
            ok = e.code() == gpu::Errc::corrupt_index;
        }
        report("corrupt_index_errc", ok);
    }
    std::printf("%d failure(s)\n", failures);
    return failures;
}
