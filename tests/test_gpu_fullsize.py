"""Parity at the BASELINE configs' full sizes (VERDICT r1 "What's weak" 1): every other image test
runs a downscaled scene. Here the GPU renders the real volumes and frames, compared at matched
per-pixel streams with
  * C2 (256^3 fBm, UNORM8, 1024^2, 16 spp, single scattering): the whole frame against the
    unmodified reference's render (oracle/_ref);
  * C3 (1024^3 turbulence, AFFINE8 and AFFINE4), C5 (the same volume with F32 leaves) and C4
    (2048^3 sparse field at 35% leaves, AFFINE8, 3840x2160, 16 spp, ratio tracking): every 64th
    16x16 tile of the full frame, against the reference's render body on the dequantised grid
    (pathtrace) or the C restatement (ratio; no reference implementation exists).
The volumes are encoded by the streaming device encoder (byte-identical to the host encoder,
tests/test_gpu_stream_encoder.py). Thresholds: the north-star relative RMSE <= 1e-3, and the
bit-identical pixel fraction measured on the B200 (FP64 tracking; CUDA's log/sincos may differ from
glibc's in the last ulp, which can flip one decision of a path)."""
import numpy as np
import pytest

import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import scenes as S
from helpers import image_parity

pytestmark = pytest.mark.gpu

STRIDE = 64


def _tile_mask(cam, stride, phase=0):
    tx = (cam.width + 15) // 16
    m = np.zeros((cam.height, cam.width), bool)
    for t in range(phase, tx * ((cam.height + 15) // 16), stride):
        y0, x0 = (t // tx) * 16, (t % tx) * 16
        m[y0:y0 + 16, x0:x0 + 16] = True
    return m


def _grid_bytes(sc):
    if sc.volume == "marschner_lobb":
        return P.compress(P.synth(sc.volume, sc.dims, sc.volume_seed), voxel_type=sc.voxel_type)[0]
    return P.synth_compress(sc.volume, sc.dims, sc.volume_seed)[0]


def _report(name, same, rmse, n):
    print(f"{name}: {n} px, identical {same:.5f}, rel RMSE {rmse:.2e}")


def test_c2_full_frame_matches_reference(gpu, ref):
    sc = S.SCENES["C2"]
    svdb = _grid_bytes(sc)
    g = P.DeviceGrid(svdb, sc.codec)
    cam = sc.camera()
    img = P.render(g, sc.tf, cam, sc.settings)
    want = ref.open(bytes(svdb)).render(sc.tf, cam, sc.settings)
    same, rmse = image_parity(img.pixels, want)
    _report("C2 full frame", same, rmse, cam.width * cam.height)
    assert rmse <= 1e-3 and same >= 0.999


@pytest.mark.parametrize("name,codec", [("C3", P.Codec.affine8), ("C3_4bit", P.Codec.affine4), ("C5", P.Codec.f32)])
def test_c3_c5_full_volume_tile_subset_matches_reference(gpu, ref, orc, name, codec):
    sc = S.SCENES[name]
    svdb = _grid_bytes(sc)
    g = P.DeviceGrid(svdb, codec)
    cam = sc.camera()
    img = P.render(g, sc.tf, cam, sc.settings)
    deq = bytes(svdb) if codec == P.Codec.f32 else orc.quantize(bytes(svdb), int(codec))[0]
    del svdb
    rg = ref.open(deq)
    rg.macrocells(sc.tf)
    want, _, paths, _ = rg.render_tiles(sc.tf, cam, sc.settings, tile_stride=STRIDE, tile_phase=0, count=False)
    m = _tile_mask(cam, STRIDE)
    same, rmse = image_parity(img.pixels[m], want[m])
    _report(f"{name} ({codec.name}) every {STRIDE}th tile", same, rmse, int(m.sum()))
    assert paths == int(m.sum()) * sc.settings.spp
    assert rmse <= 1e-3 and same >= 0.999


def test_c4_full_volume_ratio_tile_subset_matches_oracle(gpu, orc):
    sc = S.SCENES["C4"]
    svdb = _grid_bytes(sc)
    n_leaf = int(np.frombuffer(bytes(svdb[52:60]), np.uint64)[0])
    blocks = (2048 // 8) ** 3
    print(f"C4 leaves: {n_leaf} = {100 * n_leaf / blocks:.2f}% of the 8^3 blocks")
    assert abs(n_leaf / blocks - 0.35) <= 0.01  # 35% +- 1% non-background leaves
    g = P.DeviceGrid(svdb, P.Codec.affine8)
    cam = sc.camera()
    img = P.render(g, sc.tf, cam, sc.settings)
    deq = orc.quantize(bytes(svdb), int(P.Codec.affine8))[0]
    del svdb
    want, _, _ = orc.open(deq).render(sc.tf, cam, sc.settings, tile_rank=0, tile_nranks=STRIDE)
    m = _tile_mask(cam, STRIDE)
    same, rmse = image_parity(img.pixels[m], want[m])
    _report(f"C4 ratio every {STRIDE}th tile", same, rmse, int(m.sum()))
    assert rmse <= 1e-3 and same >= 0.99
