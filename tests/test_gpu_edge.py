"""Edge cases of the render path on the B200 against the unmodified reference (oracle/_ref) and the
C restatement, the way the reference's own tests probe them (test_render.cpp, test_dda.cpp):
non-cubic grids with tiles and a non-zero background, cameras inside the volume, images whose size
is not a multiple of the 16x16 tile, 1x1 frames, zero bounces / immediate Russian roulette, and
rays that never meet the grid.
"""
import numpy as np
import pytest

import paper_2504_04564_b200 as P
from helpers import MIN_IDENTICAL, SplitMix, image_parity

pytestmark = pytest.mark.gpu

RMSE_TOL = 1e-3


def _tile_grid(ref, dims=(70, 45, 33), background=0.3, seed=11):
    """Voxels, leaf-sized tiles (kind 1) over a non-cubic grid with a non-zero background."""
    r = SplitMix(seed)
    ops = []
    for _ in range(3000):
        c = (int(r.uniform() * dims[0]), int(r.uniform() * dims[1]), int(r.uniform() * dims[2]))
        ops.append((0, c, float(np.float32(r.uniform()))))
    for _ in range(40):
        o = (8 * int(r.uniform() * (dims[0] // 8)), 8 * int(r.uniform() * (dims[1] // 8)),
             8 * int(r.uniform() * (dims[2] // 8)))
        ops.append((1, o, float(np.float32(r.uniform()))))
    return ref.build_ops(dims, background, ops)


TF = P.TransferFunction(0.0, 1.0, [[0.9, 0.8, 0.7, 0.0], [0.6, 0.9, 0.8, 0.5], [0.9, 0.9, 0.9, 1.0]], 0.08)


def _check(img, want, min_same=MIN_IDENTICAL):
    same, rmse = image_parity(img, want)
    print(f"identical {same:.4f} rel RMSE {rmse:.2e}")
    assert rmse <= RMSE_TOL and same >= min_same


@pytest.mark.parametrize("codec", [P.Codec.f32, P.Codec.affine8])
@pytest.mark.parametrize("mode", [P.RenderMode.pathtrace, P.RenderMode.iso, P.RenderMode.ratio])
def test_tiles_background_noncubic(gpu, ref, orc, codec, mode):
    svdb = _tile_grid(ref)
    g = P.DeviceGrid(svdb, codec)
    src = svdb if codec == P.Codec.f32 else orc.quantize(svdb, int(codec))[0]
    cam = P.Camera(position=(140.0, 90.0, -60.0), look_at=(35.0, 22.0, 16.0), fov_y_deg=40.0, width=53, height=37)
    st = P.RenderSettings(spp=8, seed=5, mode=mode, iso_value=0.45, background_color=(0.2, 0.1, 0.05))
    img = P.render(g, TF, cam, st).pixels
    if mode == P.RenderMode.ratio:
        want, _, _ = orc.open(src).render(TF, cam, st)
    else:
        want = ref.open(src).render(TF, cam, st)
    _check(img, want)


@pytest.mark.parametrize("mode", [P.RenderMode.pathtrace, P.RenderMode.ratio, P.RenderMode.ea])
def test_camera_inside_volume(gpu, ref, orc, mode):
    svdb = _tile_grid(ref, dims=(64, 64, 64), background=0.05, seed=3)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    cam = P.Camera(position=(30.2, 33.7, 29.9), look_at=(50.0, 10.0, 60.0), fov_y_deg=70.0, width=40, height=24)
    st = P.RenderSettings(spp=6, seed=9, mode=mode)
    img = P.render(g, TF, cam, st).pixels
    if mode == P.RenderMode.pathtrace:
        want = ref.open(svdb).render(TF, cam, st)
    else:
        want, _, _ = orc.open(svdb).render(TF, cam, st)
    _check(img, want)


@pytest.mark.parametrize("wh", [(1, 1), (17, 33), (31, 16), (16, 1)])
def test_odd_image_sizes(gpu, ref, wh):
    svdb = _tile_grid(ref, dims=(40, 40, 40), seed=21)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    cam = P.Camera(position=(19.5, 19.5, -70.0), look_at=(19.5, 19.5, 19.5), width=wh[0], height=wh[1])
    st = P.RenderSettings(spp=16, seed=2)
    img = P.render(g, TF, cam, st)
    assert img.pixels.shape == (wh[1], wh[0], 3)
    assert img.stats["paths"] == wh[0] * wh[1] * 16
    _check(img.pixels, ref.open(svdb).render(TF, cam, st), min_same=0.95)


@pytest.mark.parametrize("bounces,rr", [(0, 3), (1, 0), (64, 0), (2, 1)])
def test_bounce_limits_and_roulette(gpu, ref, bounces, rr):
    # trace_path's cutoff (++bounces > max_bounces -> 0) and RR from rr_start (render.hpp:171-185)
    svdb = _tile_grid(ref, dims=(48, 48, 48), background=0.4, seed=8)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    cam = P.Camera(position=(23.5, 60.0, -50.0), look_at=(23.5, 23.5, 23.5), width=32, height=32)
    st = P.RenderSettings(spp=8, seed=13, max_bounces=bounces, rr_start_bounce=rr)
    _check(P.render(g, TF, cam, st).pixels, ref.open(svdb).render(TF, cam, st))


def test_rays_missing_the_grid_see_ambient(gpu, ref):
    svdb = _tile_grid(ref, dims=(32, 32, 32), seed=4)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    cam = P.Camera(position=(500.0, 500.0, 500.0), look_at=(900.0, 800.0, 700.0), width=16, height=16)
    st = P.RenderSettings(spp=4, ambient_radiance=(0.25, 0.5, 0.75))
    img = P.render(g, TF, cam, st).pixels
    assert np.all(img == np.array([0.25, 0.5, 0.75], np.float32))
    assert np.array_equal(img, ref.open(svdb).render(TF, cam, st))


def test_far_positions_sample_background(gpu, ref):
    # sample.hpp lattice_coord clamp at +-1e9 (test_sample.cpp:28-73: background at +-1e30)
    svdb = _tile_grid(ref, dims=(32, 32, 32), background=0.3, seed=4)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    xyz = np.array([[1e30, 0, 0], [-1e30, 5, 5], [3e9, -3e9, 1e12], [np.float64(-0.0), 0.0, 0.0]], np.float64)
    got = g.sample(xyz)
    want = ref.open(svdb).sample(xyz)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_node_walk_without_leaf_directory_is_identical(gpu, ref, monkeypatch):
    # grids whose leaf directory would exceed its budget fall back to the root/upper/lower walk
    # (SVDBGPU_NO_LEAF_DIR forces it): same voxels, samples and images bit for bit
    from helpers import all_coords, bits
    svdb = _tile_grid(ref, dims=(70, 45, 33), background=0.3, seed=11)
    with_dir = P.DeviceGrid(svdb, P.Codec.affine8)
    monkeypatch.setenv("SVDBGPU_NO_LEAF_DIR", "1")
    no_dir = P.DeviceGrid(svdb, P.Codec.affine8)
    assert no_dir.device_bytes < with_dir.device_bytes
    ijk = all_coords((-2, -2, -2), (73, 48, 36))
    assert np.array_equal(bits(with_dir.read_voxels(ijk)), bits(no_dir.read_voxels(ijk)))
    cam = P.Camera(position=(140.0, 90.0, -60.0), look_at=(35.0, 22.0, 16.0), fov_y_deg=40.0, width=53, height=37)
    for mode in (P.RenderMode.pathtrace, P.RenderMode.ratio, P.RenderMode.ea):
        st = P.RenderSettings(spp=8, seed=5, mode=mode)
        a = P.render(with_dir, TF, cam, st).pixels
        b = P.render(no_dir, TF, cam, st).pixels
        assert np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("spp,nranks", [(40, 1), (33, 1), (36, 3), (17, 2)])
def test_sample_chunked_items_match_reference(gpu, ref, spp, nranks):
    # sample-chunked work items (>= 32 spp on one GPU, any split frame): per-sample results are
    # summed in order afterwards, so frames stay bit-identical, for chunk counts that do not divide
    # spp and for spp not a multiple of 4 (scalar reduce path), on full and packed tile splits
    svdb = _tile_grid(ref, dims=(48, 40, 36), background=0.2, seed=19)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    cam = P.Camera(position=(23.5, 70.0, -60.0), look_at=(23.5, 19.5, 17.5), width=37, height=29)
    st = P.RenderSettings(spp=spp, seed=77, max_bounces=16, rr_start_bounce=2)
    want = ref.open(svdb).render(TF, cam, st)
    full = np.zeros_like(want)
    tiles_x = (cam.width + 15) // 16
    for r in range(nranks):
        img = P.render(g, TF, cam, st, tile_rank=r, tile_nranks=nranks).pixels
        for t in range(r, tiles_x * ((cam.height + 15) // 16), nranks):
            y0, x0 = (t // tiles_x) * 16, (t % tiles_x) * 16
            full[y0:y0 + 16, x0:x0 + 16] = img[y0:y0 + 16, x0:x0 + 16]
    _check(full, want)


@pytest.mark.parametrize("spp", [4, 36])
def test_packed_device_split_and_unpack_match_reference(gpu, ref, spp):
    # the multi-GPU data path on one GPU: each "rank" renders its tiles into a packed device buffer
    # (svdbgpu_render_device, packed=1; sample-chunked at 36 spp), the buffers are concatenated as the
    # NCCL gather would and k_unpack assembles the frame -> the reference's frame bit for bit
    torch = pytest.importorskip("torch")
    svdb = _tile_grid(ref, dims=(48, 40, 36), background=0.2, seed=23)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    cam = P.Camera(position=(23.5, 70.0, -60.0), look_at=(23.5, 19.5, 17.5), width=53, height=35)
    st = P.RenderSettings(spp=spp, seed=5, max_bounces=8, rr_start_bounce=2)
    want = ref.open(svdb).render(TF, cam, st)
    nranks = 3
    max_tiles = P.tiles_for_rank(cam.width, cam.height, 0, nranks)
    bufs = [torch.zeros(max_tiles * 768, dtype=torch.float32, device="cuda") for _ in range(nranks)]
    for r in range(nranks):
        P.render_device(g, TF, cam, st, bufs[r].data_ptr(), 0, packed=True, tile_rank=r, tile_nranks=nranks)
    allp = torch.cat(bufs)
    frame = torch.zeros(cam.height * cam.width * 3, dtype=torch.float32, device="cuda")
    P.unpack_tiles_device(allp.data_ptr(), nranks, max_tiles, cam.width, cam.height, frame.data_ptr(), 0)
    torch.cuda.synchronize()
    got = frame.cpu().numpy().reshape(cam.height, cam.width, 3)
    _check(got, want)


@pytest.mark.parametrize("n_entries", [1025, 4096])
@pytest.mark.parametrize("mode", [P.RenderMode.pathtrace, P.RenderMode.ratio])
def test_large_transfer_function_reads_global(gpu, ref, orc, n_entries, mode):
    # TFs above kTfSmemMax (1024) entries are read from global memory instead of shared memory; any
    # entry count the reference accepts renders (a 4096-entry LUT used to fail to launch)
    svdb = _tile_grid(ref, dims=(40, 36, 33), background=0.1, seed=31)
    r = SplitMix(n_entries)
    ent = [[r.uniform(), r.uniform(), r.uniform(), r.uniform()] for _ in range(n_entries)]
    tf = P.TransferFunction(0.0, 1.0, ent, 0.05)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    maj = g.macrocells(tf)[3]
    want_maj = ref.open(svdb).macrocells(tf)[3]
    assert np.array_equal(maj.view(np.uint32), want_maj.view(np.uint32))
    cam = P.Camera(position=(19.5, 60.0, -50.0), look_at=(19.5, 17.5, 16.0), width=24, height=20)
    st = P.RenderSettings(spp=2, seed=9, mode=mode)
    img = P.render(g, tf, cam, st).pixels
    want = (ref.open(svdb).render(tf, cam, st) if mode == P.RenderMode.pathtrace
            else orc.open(svdb).render(tf, cam, st)[0])
    _check(img, want)


def test_rank_with_no_tiles_succeeds(gpu, ref):
    # a 16x16 frame has one tile: ranks 1..3 of 4 own nothing and must render nothing, successfully
    svdb = _tile_grid(ref, dims=(24, 24, 24), background=0.0, seed=3)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    cam = P.Camera(position=(11.5, 40.0, -30.0), look_at=(11.5, 11.5, 11.5), width=16, height=16)
    st = P.RenderSettings(spp=2, seed=1)
    for r in range(1, 4):
        img = P.render(g, TF, cam, st, tile_rank=r, tile_nranks=4)
        assert img.stats["paths"] == 0
    with pytest.raises(P.Error):
        P.render(g, TF, cam, st, tile_rank=4, tile_nranks=4)


def test_render_multi_one_device_matches_render(gpu, ref):
    # the single-process multi-device entry point (svdbgpu_render_multi) on the one GPU here: device
    # split bookkeeping, packed output, k_unpack and the host copy give the render() frame bit for bit
    svdb = _tile_grid(ref, dims=(48, 40, 36), background=0.2, seed=29)
    g = P.DeviceGrid(svdb, P.Codec.f32, device=0)
    cam = P.Camera(position=(23.5, 70.0, -60.0), look_at=(23.5, 19.5, 17.5), width=53, height=35)
    for st in (P.RenderSettings(spp=4, seed=5, max_bounces=8), P.RenderSettings(spp=36, seed=6),
               P.RenderSettings(spp=3, seed=2, mode=P.RenderMode.ratio)):
        a = P.render(g, TF, cam, st)
        b = P.render_multi([g], TF, cam, st)
        assert np.array_equal(a.pixels.view(np.uint32), b.pixels.view(np.uint32))
        assert b.stats["paths"] == a.stats["paths"] and b.stats["gather_ms"] == 0.0
    want = ref.open(svdb).render(TF, cam, P.RenderSettings(spp=4, seed=5, max_bounces=8))
    _check(P.render_multi([g], TF, cam, P.RenderSettings(spp=4, seed=5, max_bounces=8)).pixels, want)
    with pytest.raises(P.Error) as e:  # one grid per device
        P.render_multi([g, g], TF, cam, P.RenderSettings(spp=1))
    assert e.value.status == P.api.E_INVALID_ARG
