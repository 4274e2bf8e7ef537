"""Quantised SVDB v2 container (svdbgpu_quantise): v1 -> v2 on the GPU codec,
v2 loads to exactly the grid the v1 bytes give with that codec, the file shrinks as the leaf
records do, and corrupt / mismatched v2 inputs fail with the reference's error classes."""
import struct

import numpy as np
import pytest

import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import scenes as S
from helpers import all_coords, bits, scene_svdb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,codec", [("C3", P.Codec.affine8), ("C3", P.Codec.affine4), ("C2", P.Codec.unorm8),
                                        ("C4", P.Codec.affine8)])
def test_v2_round_trip_is_exact(gpu, name, codec):
    sc = S.scaled(name, 16 if name != "C2" else 4, spp=4, image_factor=8)
    _, svdb, _ = scene_svdb(sc)
    q = P.quantise(svdb, codec)
    assert q[:4] == b"SVDB" and struct.unpack_from("<II", q, 4)[0] == 2
    assert struct.unpack_from("<I", q, 68)[0] == int(codec)
    g1 = P.DeviceGrid(svdb, codec)
    g2 = P.DeviceGrid(q)
    assert g2.codec == codec and g2.dims == g1.dims and g2.background == g1.background
    rec = 88 + (256 if codec == P.Codec.affine4 else 512)
    assert len(svdb) - len(q) == (2128 - rec) * g1.counts["leaf"]
    d = g1.dims
    ijk = all_coords((-1, -1, -1), (d[0] + 1, d[1] + 1, d[2] + 1))
    assert np.array_equal(bits(g1.read_voxels(ijk)), bits(g2.read_voxels(ijk)))
    cam = sc.camera()
    a = P.render(g1, sc.tf, cam, sc.settings).pixels
    b = P.render(g2, sc.tf, cam, sc.settings).pixels
    assert np.array_equal(bits(a), bits(b))


def test_v2_errors(gpu):
    sc = S.scaled("C3", 16, spp=1, image_factor=8)
    _, svdb, _ = scene_svdb(sc)
    q = P.quantise(svdb, P.Codec.affine8)
    with pytest.raises(P.Error):          # truncated
        P.DeviceGrid(q[:-8])
    bad = bytearray(q)
    struct.pack_into("<I", bad, 68, 9)    # unknown codec word
    with pytest.raises(P.Error):
        P.DeviceGrid(bytes(bad))
    bad = bytearray(q)
    struct.pack_into("<I", bad, 4, 3)     # unknown version
    with pytest.raises(P.Error) as e:
        P.DeviceGrid(bytes(bad))
    assert e.value.code == P.Errc.version_mismatch
    with pytest.raises(P.Error):          # a v2 file keeps its codec
        P.DeviceGrid(q, P.Codec.f32)
    with pytest.raises(P.Error):          # quantise reads v1 only
        P.quantise(q, P.Codec.affine8)
