"""CPU: the C restatement (oracle/liboracle.so) is pinned against the reference's golden vectors
(tests/golden, generated from the unmodified reference) and, where the reference build exists,
against the reference itself on fresh randomized cases. Also known-answer tests for the
north-star additions the reference lacks (codec, EA, ratio tracking)."""
import os

import numpy as np
import pytest

import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import scenes as S
from helpers import SplitMix, all_coords, bits, image_parity, mixed_tile_ops, random_voxel_ops, scene_svdb

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def _gold_scene(gold):
    tf = P.TransferFunction(0.0, 1.0, gold["tf_entries"], 0.5)
    c = gold["cam"]
    cam = P.Camera(position=tuple(c[0:3]), look_at=tuple(c[3:6]), up=tuple(c[6:9]), fov_y_deg=float(c[9]),
                   width=int(c[10]), height=int(c[11]))
    return tf, cam


def test_oracle_matches_golden_lookups(orc, gold):
    g = orc.open(gold["voxels_svdb"].tobytes())
    for cached in (False, True):
        assert np.array_equal(bits(g.read_voxels(gold["voxels_coords"], cached)), bits(gold["voxels_values"]))
    g2 = orc.open(gold["tiles_svdb"].tobytes())
    assert np.array_equal(bits(g2.read_voxels(gold["tiles_coords"], True)), bits(gold["tiles_values"]))
    gm = orc.open(gold["ml_svdb"].tobytes())
    assert np.array_equal(bits(gm.sample(gold["ml_points"], 1)), bits(gold["ml_trilinear"]))
    assert np.array_equal(bits(gm.sample(gold["ml_points"], 0)), bits(gold["ml_nearest"]))


def test_oracle_matches_golden_macrocells_and_images(orc, gold):
    gm = orc.open(gold["ml_svdb"].tobytes())
    tf, cam = _gold_scene(gold)
    cells, cmin, cmax, maj, empty = gm.macrocells(tf)
    assert list(cells) == list(gold["ml_cells"])
    for a, b in ((cmin, "ml_cmin"), (cmax, "ml_cmax"), (maj, "ml_maj")):
        assert np.array_equal(bits(a), bits(gold[b]))
    assert np.array_equal(empty, gold["ml_empty"])
    img, _, _ = gm.render(tf, cam, P.RenderSettings(spp=4, max_bounces=64, rr_start_bounce=3, seed=11))
    assert np.array_equal(bits(img), bits(gold["pt_image"]))
    iso, _, _ = gm.render(tf, cam, P.RenderSettings(spp=1, seed=3, mode=P.RenderMode.iso, iso_value=0.55,
                                                    background_color=(0.1, 0.2, 0.3)))
    assert np.array_equal(bits(iso), bits(gold["iso_image"]))


def test_rng_streams_golden(orc, gold):
    keys = [(0, 0, 0, 0), (11, 5, 7, 3), (2 ** 63 + 5, -1, 4096, 63)]
    for (s, px, py, k), want in zip(keys, gold["rng"]):
        assert np.array_equal(orc.rng_uniforms(s, px, py, k, 8), want)
        # and the Python SplitMix used to build the randomized test streams
        h = SplitMix.mix64(s)
        h = SplitMix.mix64(h ^ (((px & 0xFFFFFFFF) << 32) | (py & 0xFFFFFFFF)))
        h = SplitMix.mix64(h ^ (k & 0xFFFFFFFF))
        r = SplitMix(0)
        r.state = SplitMix.mix64(h)
        assert np.array_equal(np.array([r.uniform() for _ in range(8)]), want)


def test_encoder_reproduces_golden_svdb(gold):
    vol = gold["ml_volume"]
    mine, _ = P.compress(vol, P.CompressionParams(1.0), voxel_type=P.VoxelType.u8)
    assert mine == gold["ml_svdb"].tobytes()
    import hashlib
    half, _ = P.compress(vol, P.CompressionParams(0.5), voxel_type=P.VoxelType.u8)
    assert hashlib.sha256(half).digest() == gold["ml_half_svdb_sha256"].tobytes()


# ---- against the live reference build (when present) ----
def test_oracle_vs_reference_randomized(orc, ref):
    ops, r = random_voxel_ops(99, 3000, 96)
    svdb = ref.build_ops((96, 96, 200), 0.25, ops + [(1, (16, 16, 16), 3.0), (2, (0, 0, 128), 1.0)])
    q = np.array([[int(r.uniform() * 140) - 12 for _ in range(3)] for _ in range(50000)], np.int32)
    og, rg = orc.open(svdb), ref.open(svdb)
    for cached in (False, True):
        assert np.array_equal(bits(og.read_voxels(q, cached)), bits(rg.read_voxels(q, cached)))
    p = np.random.default_rng(3).uniform(-10, 110, size=(50000, 3))
    for mode in (0, 1):
        assert np.array_equal(bits(og.sample(p, mode)), bits(rg.sample(p, mode)))


@pytest.mark.parametrize("name,factor,mode", [("C1", 1, "pathtrace"), ("C2", 8, "pathtrace"), ("C3", 16, "pathtrace"),
                                              ("C1", 1, "iso")])
def test_oracle_render_bit_exact_vs_reference(orc, ref, name, factor, mode):
    sc = S.scaled(name, factor, spp=2, image_factor=8, mode=P.RenderMode[mode])
    st = sc.settings
    if mode == "iso":
        st = P.RenderSettings(spp=1, seed=5, mode=P.RenderMode.iso, iso_value=0.6)
    _, svdb, _ = scene_svdb(sc)
    cam = sc.camera()
    want = ref.open(svdb).render(sc.tf, cam, st)
    got, lk, pa = orc.open(svdb).render(sc.tf, cam, st)
    assert np.array_equal(bits(got), bits(want))
    assert pa == cam.width * cam.height * st.spp


def test_oracle_macrocells_vs_reference(orc, ref):
    sc = S.scaled("C2", 4)
    _, svdb, _ = scene_svdb(sc, quality=0.5)
    a = orc.open(svdb).macrocells(sc.tf)
    b = ref.open(svdb).macrocells(sc.tf)
    assert a[0] == b[0]
    for x, y in zip(a[1:4], b[1:4]):
        assert np.array_equal(bits(x), bits(y))
    assert np.array_equal(a[4], b[4])


# ---- north-star additions (no reference implementation: analytic / property pins) ----
def test_unorm8_device_decode_identity():
    # the device decodes UNORM8 as float((double)k * (1.0/255.0)); it equals k/255.0f for all k
    k = np.arange(256)
    want = (k.astype(np.float32) / np.float32(255.0)).astype(np.float32)
    got = (k.astype(np.float64) * (1.0 / 255.0)).astype(np.float32)
    assert np.array_equal(bits(got), bits(want))


@pytest.mark.parametrize("codec", [1, 2, 3])
def test_codec_properties(orc, codec):
    sc = S.scaled("C2" if codec == 1 else "C3", 8)
    vol, svdb, _ = scene_svdb(sc)
    deq, codes, params = orc.quantize(svdb, codec)
    og, dg = orc.open(svdb), orc.open(deq)
    c = all_coords((0, 0, 0), sc.dims)
    a, b = og.read_voxels(c), dg.read_voxels(c)
    if codec == 1:
        assert np.array_equal(bits(a), bits(b))  # u8 sources: exact
    else:
        levels = 255 if codec == 2 else 15
        assert codes.max() <= levels
        assert np.abs(a.astype(np.float64) - b).max() <= params[:, 1].max() * 0.5 * (1 + 1e-6) + 1e-7
        # leaf decode is exactly fmaf(code, scale, lo)
        dec = np.array([orc.lib.so_decode(codec, int(cc), float(lo), float(s))
                        for cc, (lo, s) in zip(codes[:50, 7], params[:50])], np.float32)
        ref = (np.float64(1.0) * codes[:50, 7] * params[:50, 1].astype(np.float64) + params[:50, 0]).astype(np.float32)
        assert np.allclose(dec, ref, rtol=0, atol=1e-6)


def test_constant_leaf_quantises_exactly(orc, ref):
    # a fully constant leaf gets scale 0 and decodes to its value exactly
    ops = [(0, (x, y, z), 0.375) for z in range(8) for y in range(8) for x in range(8)] + [(0, (9, 9, 9), 2.0)]
    svdb = ref.build_ops((32, 32, 32), 0.0, ops)
    deq, codes, params = orc.quantize(svdb, 2)
    assert np.array_equal(bits(orc.open(deq).read_voxels(all_coords((0, 0, 0), (8, 8, 8)))),
                          bits(np.full(512, 0.375, np.float32)))


def test_ratio_and_delta_estimators_agree_in_homogeneous_cube(orc, ref):
    # same integral, two estimators: delta-tracking escape vs ratio-tracked transmittance
    svdb = ref.build_ops((32, 32, 32), 1.0, [])
    tf = P.TransferFunction(0.0, 2.0, [[0.9, 0.9, 0.9, 1.0]] * 2, 0.06)
    cam = P.Camera(position=(15.5, 15.5, -90.0), look_at=(15.5, 15.5, 15.5), fov_y_deg=25.0, width=24, height=24)
    og = orc.open(svdb)
    d, _, _ = og.render(tf, cam, P.RenderSettings(spp=256, seed=1, mode=P.RenderMode.pathtrace))
    r, _, _ = og.render(tf, cam, P.RenderSettings(spp=256, seed=2, mode=P.RenderMode.ratio))
    assert abs(d.mean() - r.mean()) < 0.006
    assert r.std() <= d.std() * 1.05  # ratio tracking never noisier here


@pytest.mark.parametrize("cell", [8, 128])
def test_node_majorant_grids_are_unbiased(orc, cell):
    # delta tracking is unbiased for any bounding majorant: leaf (8^3) and lower-node (128^3)
    # majorant grids estimate the same image as the reference's 32^3 macrocells, with fewer
    # lookups for the tighter grid
    sc = S.scaled("C3", 16, spp=32, image_factor=16)
    _, svdb, _ = scene_svdb(sc)
    og = orc.open(svdb)
    cam = sc.camera()
    base, lk32, _ = og.render(sc.tf, cam, P.RenderSettings(spp=32, seed=1, max_bounces=64, rr_start_bounce=3))
    img, lk, _ = og.render(sc.tf, cam, P.RenderSettings(spp=32, seed=1, max_bounces=64, rr_start_bounce=3,
                                                         majorant_cell=cell))
    assert abs(img.mean() - base.mean()) < 3e-3
    assert (lk < lk32) if cell == 8 else (lk >= lk32)
    with pytest.raises(RuntimeError):
        og.render(sc.tf, cam, P.RenderSettings(spp=1, majorant_cell=16))


def test_ea_transmittance_is_beer_lambert(orc, ref):
    # EA through a homogeneous slab: T = exp(-sigma * L) up to the dt discretisation (exact here:
    # a = 1 - exp(-sigma dt) compounds to exp(-sigma * n dt))
    svdb = ref.build_ops((65, 65, 65), 1.0, [])
    sigma = 0.02
    tf = P.TransferFunction(0.0, 2.0, [[0.0, 0.0, 0.0, 1.0]] * 2, sigma)
    cam = P.Camera(position=(32.0, 32.0, -100.0), look_at=(32.0, 32.0, 32.0), fov_y_deg=1.0, width=4, height=4)
    og = orc.open(svdb)
    st = P.RenderSettings(spp=1, seed=4, mode=P.RenderMode.ea, ea_step=0.5, ea_min_transmittance=0.0,
                          background_color=(1.0, 1.0, 1.0))
    img, _, _ = og.render(tf, cam, st)
    # ray length through the box ~64 voxels; n = 128 samples of dt 0.5 (+/- one at the ends)
    assert np.all(np.abs(img[..., 0] - np.exp(-sigma * 64.0)) < 0.02)


def test_hdda_in_one_lower_node_region_is_the_flat_dda(orc):
    # a grid inside one 128^3 lower-node region: the coarse DDA visits that single region over the
    # clipped segment and the majorant-grid DDA restarts at its entry -> exactly the flat traversal
    sc = S.scaled("C3", 16, spp=4, image_factor=16)
    _, svdb, _ = scene_svdb(sc)
    og = orc.open(svdb)
    cam = sc.camera()
    for mode in (P.RenderMode.pathtrace, P.RenderMode.ratio):
        st = P.RenderSettings(spp=4, seed=3, mode=mode)
        a, _, _ = og.render(sc.tf, cam, st)
        b, _, _ = og.render(sc.tf, cam, P.RenderSettings(spp=4, seed=3, mode=mode, hdda=1))
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("mode", [P.RenderMode.pathtrace, P.RenderMode.ratio])
def test_hdda_skips_empty_regions_without_bias(orc, mode):
    # the sparse C4 field at 256^3 (2 x 2 x 2 lower-node regions, some without draws): skipping a
    # region in one step changes where the majorant-grid DDA restarts, not the estimator
    sc = S.scaled("C4", 8, spp=64, image_factor=40)
    _, svdb, _ = scene_svdb(sc)
    og = orc.open(svdb)
    cam = sc.camera()
    st = dict(spp=64, seed=11, max_bounces=64, rr_start_bounce=3, mode=mode)
    flat, _, _ = og.render(sc.tf, cam, P.RenderSettings(**st))
    hier, _, _ = og.render(sc.tf, cam, P.RenderSettings(**st, hdda=1))
    assert abs(hier.mean() - flat.mean()) < 4e-3
    with pytest.raises(RuntimeError):  # the coarse level is the lower node: majorant cells must be finer
        og.render(sc.tf, cam, P.RenderSettings(spp=1, majorant_cell=128, hdda=1))
