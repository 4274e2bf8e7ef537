"""K4/K5/K6 + ISO parity on the B200 against the CPU oracles at matched per-pixel RNG streams.

* pathtrace / iso: the UNMODIFIED reference render() (oracle/_ref) is the image oracle; for
  quantised grids it renders the dequantised SVDB of the same topology.
* ea / ratio: no reference implementation exists; the C restatement (oracle/liboracle.so) is
  the oracle.
Tolerance (BASELINE.json north_star): per-image relative RMSE <= 1e-3 at matched streams and spp.
FP64 libm (log/sin/cos/exp) differs from glibc by <= 1-2 ulp, so a few pixels may differ in the
last bits; we also require the bulk of pixels to be bit-identical.
"""
import numpy as np
import pytest

import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import scenes as S
from helpers import MIN_IDENTICAL, image_parity, scene_svdb

pytestmark = pytest.mark.gpu

RMSE_TOL = 1e-3


def _render_pair(ref_like, gpu_grid, sc, settings=None, cam=None):
    st = settings or sc.settings
    cam = cam or sc.camera()
    img = P.render(gpu_grid, sc.tf, cam, st)
    want = ref_like(sc.tf, cam, st)
    return img, want


@pytest.mark.parametrize("name,factor,spp,bounces", [
    ("C1", 1, 4, 64),       # u8 ML, UNORM8, multi-bounce
    ("C2", 4, 8, 1),        # u8 smoke, UNORM8, single scattering (C2's integrator)
    ("C3", 16, 4, 64),      # f32 turbulence, F32 leaves (reference layout, C5)
])
def test_pathtrace_matches_reference(gpu, ref, name, factor, spp, bounces):
    sc = S.scaled(name, factor, spp=spp, image_factor=max(4, factor), mode=P.RenderMode.pathtrace)
    st = P.RenderSettings(spp=spp, max_bounces=bounces, rr_start_bounce=3, seed=sc.settings.seed)
    _, svdb, _ = scene_svdb(sc)
    codec = P.Codec.f32 if name == "C3" else P.Codec.auto8
    g = P.DeviceGrid(svdb, codec)
    rg = ref.open(svdb)
    img, want = _render_pair(lambda tf, cam, s: rg.render(tf, cam, s), g, sc, st)
    same, rmse = image_parity(img.pixels, want)
    print(f"{name}: identical pixels {same:.4f}, rel RMSE {rmse:.2e}, stats {img.stats}")
    assert rmse <= RMSE_TOL
    assert same >= MIN_IDENTICAL
    assert img.stats["paths"] == sc.width * sc.height * spp


@pytest.mark.parametrize("codec", [P.Codec.affine8, P.Codec.affine4])
def test_pathtrace_quantised_matches_reference_on_dequantised_grid(gpu, ref, orc, codec):
    sc = S.scaled("C3", 16, spp=4, image_factor=8)
    _, svdb, _ = scene_svdb(sc)
    deq, _, _ = orc.quantize(svdb, int(codec))
    g = P.DeviceGrid(svdb, codec)
    rg = ref.open(deq)
    img, want = _render_pair(lambda tf, cam, s: rg.render(tf, cam, s), g, sc)
    same, rmse = image_parity(img.pixels, want)
    print(f"{codec.name}: identical {same:.4f} rmse {rmse:.2e}")
    assert rmse <= RMSE_TOL and same >= MIN_IDENTICAL


def test_iso_matches_reference(gpu, ref):
    sc = S.scaled("C1", 1, spp=2, image_factor=4)
    st = P.RenderSettings(spp=2, seed=7, mode=P.RenderMode.iso, iso_value=0.55,
                          background_color=(0.1, 0.2, 0.3))
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb)
    rg = ref.open(svdb)
    img, want = _render_pair(lambda tf, cam, s: rg.render(tf, cam, s), g, sc, st)
    same, rmse = image_parity(img.pixels, want)
    assert rmse <= RMSE_TOL and same >= 0.99


def test_ea_matches_oracle_c1(gpu, orc):
    sc = S.SCENES["C1"]  # the full C1 workload: 64^3 ML, 512x512 EA, 1 spp
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb)
    og = orc.open(svdb)
    img, (want, _, _) = _render_pair(lambda tf, cam, s: og.render(tf, cam, s), g, sc)
    same, rmse = image_parity(img.pixels, want)
    print(f"EA C1: identical {same:.4f} rmse {rmse:.2e}")
    assert rmse <= RMSE_TOL and same >= 0.95


def test_ratio_matches_oracle(gpu, orc):
    sc = S.scaled("C4", 32, spp=4, image_factor=16)
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb, P.Codec.affine8)
    deq, _, _ = orc.quantize(svdb, int(P.Codec.affine8))
    og = orc.open(deq)
    img, (want, _, _) = _render_pair(lambda tf, cam, s: og.render(tf, cam, s), g, sc)
    same, rmse = image_parity(img.pixels, want)
    print(f"ratio: identical {same:.4f} rmse {rmse:.2e}")
    assert rmse <= RMSE_TOL and same >= MIN_IDENTICAL


def test_ratio_and_delta_agree_statistically(gpu):
    # same scene, different estimators of the same integral: image means agree within noise
    sc = S.scaled("C4", 32, spp=64, image_factor=30)
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb, P.Codec.affine8)
    cam = sc.camera()
    a = P.render(g, sc.tf, cam, P.RenderSettings(spp=64, seed=11, mode=P.RenderMode.ratio)).pixels
    b = P.render(g, sc.tf, cam, P.RenderSettings(spp=64, seed=12, mode=P.RenderMode.pathtrace)).pixels
    assert abs(a.mean() - b.mean()) < 0.01 * max(b.mean(), 1e-3) + 3e-3


@pytest.mark.parametrize("cell", [8, 128])
@pytest.mark.parametrize("mode", [P.RenderMode.pathtrace, P.RenderMode.ratio])
def test_node_majorant_grid_matches_oracle(gpu, orc, cell, mode):
    # leaf / lower-node majorant grids: same streams as the oracle at the same cell size
    sc = S.scaled("C3", 16, spp=4, image_factor=8, mode=mode)
    st = P.RenderSettings(spp=4, seed=5, max_bounces=64, rr_start_bounce=3, mode=mode, majorant_cell=cell)
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb, P.Codec.affine8)
    deq, _, _ = orc.quantize(svdb, int(P.Codec.affine8))
    og = orc.open(deq)
    img, (want, lookups, _) = _render_pair(lambda tf, cam, s: og.render(tf, cam, s), g, sc, st)
    same, rmse = image_parity(img.pixels, want)
    print(f"cell {cell} {mode.name}: identical {same:.4f} rmse {rmse:.2e}")
    assert rmse <= RMSE_TOL and same >= MIN_IDENTICAL
    if mode == P.RenderMode.pathtrace:
        assert abs(img.stats["lookups"] - lookups) <= 1e-3 * lookups


def test_node_majorant_grid_is_unbiased_at_scale(gpu):
    # 256^3 turbulence: 8^3 / 128^3 majorant grids vs the reference's 32^3 macrocells, image means
    sc = S.scaled("C3", 4, spp=16, image_factor=8)
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb, P.Codec.affine8)
    cam = sc.camera()
    means = {}
    for cell in (32, 8, 128):
        st = P.RenderSettings(spp=16, seed=21, max_bounces=64, rr_start_bounce=3, majorant_cell=cell)
        img = P.render(g, sc.tf, cam, st)
        means[cell] = (img.pixels.mean(), img.stats["lookups"])
    print(means)
    for cell in (8, 128):
        assert abs(means[cell][0] - means[32][0]) < 3e-3
    assert means[8][1] < means[32][1]
    with pytest.raises(P.Error):
        P.render(g, sc.tf, cam, P.RenderSettings(spp=1, majorant_cell=16))


def test_tile_split_is_bit_identical(gpu):
    # GPU-count invariance (test_render.cpp:296-322 pins thread counts the same way):
    # interleaved tiles rendered as 3 "ranks" and reassembled equal the 1-rank frame bit for bit
    sc = S.scaled("C2", 8, spp=4, image_factor=6)
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb)
    cam = sc.camera()
    full = P.render(g, sc.tf, cam, sc.settings).pixels
    parts = np.zeros_like(full)
    for r in range(3):
        img = P.render(g, sc.tf, cam, sc.settings, tile_rank=r, tile_nranks=3)
        tiles_x = (cam.width + 15) // 16
        for t in range(r, tiles_x * ((cam.height + 15) // 16), 3):
            y0, x0 = (t // tiles_x) * 16, (t % tiles_x) * 16
            parts[y0:y0 + 16, x0:x0 + 16] = img.pixels[y0:y0 + 16, x0:x0 + 16]
    assert np.array_equal(full.view(np.uint32), parts.view(np.uint32))


def test_empty_scene_is_ambient(gpu, ref):
    # TracePath.EmptySceneIsAmbientEverywhere (test_render.cpp:128-146)
    g = P.DeviceGrid(ref.build_ops((64, 64, 64), 0.0, []))
    tf = P.TransferFunction(0.0, 1.0, [[1, 1, 1, 0], [1, 1, 1, 1]], 2.0)
    cam = P.Camera(position=(31.5, 31.5, -150.0), look_at=(31.5, 31.5, 31.5), width=24, height=24)
    img = P.render(g, tf, cam, P.RenderSettings(spp=8))
    assert np.all(img.pixels == 1.0)


def test_homogeneous_cube_matches_independent_mc(gpu, ref):
    # TracePath.MatchesIndependentHomogeneousReference (test_render.cpp:169-271), both integrators
    g = P.DeviceGrid(ref.build_ops((32, 32, 32), 1.0, []))
    sigma, albedo = 0.06, 0.9
    tf = P.TransferFunction(0.0, 2.0, [[albedo] * 3 + [1.0]] * 2, sigma)
    cam = P.Camera(position=(15.5, 15.5, -90.0), look_at=(15.5, 15.5, 15.5), fov_y_deg=25.0,
                   width=48, height=48)
    rng = np.random.default_rng(4242)
    n = 400000
    tan_half = np.tan(np.radians(25.0) / 2)
    px = (rng.integers(0, 48, n) + rng.random(n)) / 48
    py = (rng.integers(0, 48, n) + rng.random(n)) / 48
    d = np.stack([(2 * px - 1) * tan_half, (1 - 2 * py) * tan_half, np.ones(n)], 1)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = np.tile([15.5, 15.5, -90.0], (n, 1))
    L = np.zeros(n); tp = np.ones(n); alive = np.ones(n, bool); bounces = np.zeros(n, int)
    lo, hi = np.zeros(3), np.full(3, 31.0)
    for _ in range(200):
        if not alive.any():
            break
        inv = 1.0 / np.where(d == 0, 1e-300, d)
        ta = (lo - o) * inv; tb = (hi - o) * inv
        t0 = np.maximum(np.minimum(ta, tb).max(1), 0.0); t1 = np.maximum(ta, tb).min(1)
        hit = alive & (t1 > t0)
        fl = -np.log(1 - rng.random(n)) / sigma
        esc = alive & (~hit | (t0 + fl >= t1))
        L[esc] = tp[esc]; alive &= ~esc
        bounces[alive] += 1
        dead = alive & (bounces > 64); alive &= ~dead
        tp[alive] *= albedo
        o[alive] = o[alive] + d[alive] * (t0 + fl)[alive, None]
        z = 1 - 2 * rng.random(n); phi = 2 * np.pi * rng.random(n); r = np.sqrt(np.maximum(0, 1 - z * z))
        nd = np.stack([r * np.cos(phi), r * np.sin(phi), z], 1)
        d[alive] = nd[alive]
        rr = alive & (bounces >= 3)
        surv = np.clip(tp, 0.05, 0.95)
        kill = rr & (rng.random(n) >= surv)
        alive &= ~kill
        tp[rr & alive] /= surv[rr & alive]
    ref_mean, ref_se = L.mean(), L.std() / np.sqrt(n)
    for mode in (P.RenderMode.pathtrace, P.RenderMode.ratio):
        img = P.render(g, tf, cam, P.RenderSettings(spp=256, seed=99, mode=mode))
        ours = img.pixels[..., 0].mean()
        assert abs(ours - ref_mean) < 3 * ref_se + 0.004, (mode, ours, ref_mean)


@pytest.mark.parametrize("cell", [32, 8])
@pytest.mark.parametrize("mode", [P.RenderMode.pathtrace, P.RenderMode.ratio])
def test_hdda_matches_oracle_on_multi_region_grid(gpu, orc, cell, mode):
    # hierarchical DDA (a23): 128^3 lower-node regions without draws skipped in one step, the
    # majorant grid walked inside the others. Sparse C4 field at 256^3 (8 regions) and 512^3 (64): the
    # GPU consumes the same streams as the oracle's flight_next, visit for visit. Region entries fix
    # the first majorant cell on the entry face's axis, so a last-ulp difference in a scattered
    # direction (CUDA's sincos vs glibc) cannot move the restart; with max_bounces 0 no direction is
    # drawn at all.
    for factor, imf in ((8, 32), (4, 48)):
        _, svdb, _ = scene_svdb(S.scaled("C4", factor, spp=4, image_factor=imf, mode=mode))
        g = P.DeviceGrid(svdb, P.Codec.affine8)
        deq, _, _ = orc.quantize(svdb, int(P.Codec.affine8))
        og = orc.open(deq)
        for bounces, spp, imf2, min_same in ((0, 4, imf, 0.9999), (64, 16, imf // 2, 0.99)):
            sc = S.scaled("C4", factor, spp=spp, image_factor=imf2, mode=mode)
            st = P.RenderSettings(spp=spp, seed=7, max_bounces=bounces, rr_start_bounce=3, mode=mode,
                                  majorant_cell=cell, hdda=1)
            img, (want, lookups, _) = _render_pair(lambda tf, cam, s: og.render(tf, cam, s), g, sc, st)
            same, rmse = image_parity(img.pixels, want)
            print(f"{sc.dims[0]}^3 cell {cell} {mode.name} bounces {bounces}: identical {same:.5f} rmse {rmse:.2e}")
            assert rmse <= RMSE_TOL and same >= min_same
            if mode == P.RenderMode.pathtrace and bounces == 0:
                assert abs(img.stats["lookups"] - lookups) <= 1e-4 * lookups


def test_hdda_is_unbiased_and_validated(gpu):
    sc = S.scaled("C4", 4, spp=16, image_factor=16)
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb, P.Codec.affine8)
    cam = sc.camera()
    base = P.render(g, sc.tf, cam, P.RenderSettings(spp=16, seed=3, mode=P.RenderMode.ratio))
    hier = P.render(g, sc.tf, cam, P.RenderSettings(spp=16, seed=3, mode=P.RenderMode.ratio, hdda=1))
    assert abs(hier.pixels.mean() - base.pixels.mean()) < 3e-3
    for bad in (dict(majorant_cell=128, hdda=1), dict(precision=2, hdda=1), dict(mode=P.RenderMode.ea, hdda=1)):
        with pytest.raises(P.Error):
            P.render(g, sc.tf, cam, P.RenderSettings(spp=1, **bad))
