"""FP32-arithmetic tracking kernels (csrc/render_fast.cu: SVDBGPU_PRECISION_MIXED = FP64 geometry
+ FP32 step / sampler / TF, and SVDBGPU_PRECISION_FP32) against the reference-exact FP64 path at
matched per-pixel streams and spp.

The FP64 images are themselves pinned bit for bit to the unmodified reference / the C oracle
(test_gpu_render.py), so this is the north-star tolerance check for the FP32 path: relative RMSE
<= 1e-3 (BASELINE.json north_star), and far below the Monte Carlo noise of an independent seed.
"""
from dataclasses import replace

import pytest

import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import scenes as S
from helpers import image_parity, scene_svdb

pytestmark = pytest.mark.gpu

RMSE_TOL = 1e-3


@pytest.mark.parametrize("precision", [2, 1])
@pytest.mark.parametrize("name,factor,image_factor,spp,codec", [
    ("C3", 16, 8, 64, P.Codec.affine8),   # 64^3 turbulence, multi-bounce
    ("C3", 4, 4, 16, P.Codec.affine8),    # 256^3, 480x270
    ("C3", 16, 8, 16, P.Codec.affine4),
    ("C3", 16, 8, 16, P.Codec.f32),
    ("C2", 4, 4, 16, P.Codec.auto8),      # single scattering, u8 smoke
    ("C4", 32, 16, 16, P.Codec.affine8),  # ratio tracking, sparse
])
def test_fp32_matches_fp64_within_tolerance(gpu, name, factor, image_factor, spp, codec, precision):
    sc = S.scaled(name, factor, spp=spp, image_factor=image_factor)
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb, codec)
    cam = sc.camera()
    st = replace(sc.settings, spp=spp)
    ref = P.render(g, sc.tf, cam, st)
    fast = P.render(g, sc.tf, cam, replace(st, precision=precision))
    other = P.render(g, sc.tf, cam, replace(st, seed=st.seed + 1)).pixels
    _, rmse = image_parity(fast.pixels, ref.pixels)
    _, noise = image_parity(other, ref.pixels)
    print(f"{name} x{factor} {codec.name} spp {spp} precision {precision}: rel RMSE {rmse:.2e}, "
          f"other-seed {noise:.2e}")
    assert rmse <= RMSE_TOL
    assert rmse <= 0.02 * noise
    assert fast.stats["paths"] == ref.stats["paths"]
    assert abs(fast.stats["samples"] - ref.stats["samples"]) <= 2e-3 * ref.stats["samples"]


def test_fp32_tile_split_is_bit_identical(gpu):
    # per-pixel stream keying holds in FP32 too: 2-rank interleaved tiles == 1-rank frame
    sc = S.scaled("C2", 8, spp=4, image_factor=6)
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb)
    cam = sc.camera()
    st = replace(sc.settings, precision=2)
    full = P.render(g, sc.tf, cam, st).pixels
    tiles_x = (cam.width + 15) // 16
    for r in range(2):
        img = P.render(g, sc.tf, cam, st, tile_rank=r, tile_nranks=2).pixels
        for t in range(r, tiles_x * ((cam.height + 15) // 16), 2):
            y0, x0 = (t // tiles_x) * 16, (t % tiles_x) * 16
            assert (img[y0:y0 + 16, x0:x0 + 16] == full[y0:y0 + 16, x0:x0 + 16]).all()


def test_fp32_rejects_unsupported_modes(gpu):
    sc = S.scaled("C1", 2, spp=1, image_factor=8)
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb)
    for st in (replace(sc.settings, precision=1, mode=P.RenderMode.ea),
               replace(sc.settings, precision=1, mode=P.RenderMode.pathtrace, kernel=1),
               replace(sc.settings, precision=7)):
        with pytest.raises(P.Error):
            P.render(g, sc.tf, sc.camera(), st)
