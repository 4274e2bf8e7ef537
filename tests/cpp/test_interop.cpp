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
