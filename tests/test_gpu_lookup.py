"""K0/K1/K2/K3 parity on the B200: device layout + codec, read_voxel, sampler, macrocells.
Bit-exact against the unmodified reference (oracle/_ref) or, for the new codecs, the C oracle.
Mirrors test_tree.cpp / test_sample.cpp / test_macrocell.cpp / test_io.cpp."""
import numpy as np
import pytest

import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import scenes as S
from helpers import SplitMix, all_coords, bits, mixed_tile_ops, random_voxel_ops, scene_svdb

pytestmark = pytest.mark.gpu


def test_randomized_voxels_bit_exact(gpu, ref):
    # test_tree.cpp:160-182: 5000 random voxels, 1e5 random reads incl. out of bounds
    ops, r = random_voxel_ops()
    svdb = ref.build_ops((64, 64, 64), 0.5, ops)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    q = np.array([[int(r.uniform() * 80) - 8 for _ in range(3)] for _ in range(100000)], np.int32)
    assert np.array_equal(bits(g.read_voxels(q)), bits(ref.open(svdb).read_voxels(q)))


@pytest.mark.parametrize("prune", [False, True])
def test_mixed_tiles_every_voxel(gpu, ref, prune):
    # test_tree.cpp:184-217: lower-slot tiles + voxels, every coordinate of [-1, 64]^3
    svdb = ref.build_ops((64, 64, 64), 0.0, mixed_tile_ops(), prune=prune)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    c = all_coords((-1, -1, -1), (65, 65, 65))
    assert np.array_equal(bits(g.read_voxels(c)), bits(ref.open(svdb).read_voxels(c)))


def test_upper_tiles_and_empty_grid(gpu, ref):
    ops = [(2, (128, 0, 128), 6.0), (0, (3, 4, 5), 1.5), (1, (16, 16, 16), 3.0), (2, (0, 128, 0), 2.0)]
    svdb = ref.build_ops((300, 300, 300), 0.125, ops)
    g = P.DeviceGrid(svdb, P.Codec.f32)
    rr = SplitMix(99)
    q = np.array([[int(rr.uniform() * 340) - 20 for _ in range(3)] for _ in range(200000)], np.int32)
    assert np.array_equal(bits(g.read_voxels(q)), bits(ref.open(svdb).read_voxels(q)))
    empty = ref.build_ops((32, 32, 32), 1.25, [])  # Freeze.EmptyBuilderIsHeaderOnly
    ge = P.DeviceGrid(empty, P.Codec.f32)
    assert list(ge.read_voxels([[0, 0, 0], [31, 31, 31], [-5, 0, 0]])) == [1.25, 1.25, 1.25]


@pytest.mark.parametrize("name,factor", [("C1", 1), ("C2", 4)])
def test_u8_sources_unorm8_bit_exact_vs_reference(gpu, ref, name, factor):
    # 8-bit leaves of u8 sources decode bit-exactly to the reference tree itself
    sc = S.scaled(name, factor)
    vol, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb, P.Codec.auto8)
    assert g.codec == P.Codec.unorm8
    d = sc.dims
    c = all_coords((-2, -2, -2), (d[0] + 2, d[1] + 2, d[2] + 2))
    assert np.array_equal(bits(g.read_voxels(c)), bits(ref.open(svdb).read_voxels(c)))
    # 512 codes + 217-entry apron (padded to 256) + 8 x (lo, scale) per leaf
    assert g.leaf_payload_bytes == g.counts["leaf"] * (512 + 256 + 64)


@pytest.mark.parametrize("codec", [P.Codec.affine8, P.Codec.affine4])
def test_affine_codec_bit_exact_vs_restated_codec(gpu, orc, ref, codec):
    sc = S.scaled("C3", 16)
    vol, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb, codec)
    deq, codes, params = orc.quantize(svdb, int(codec))
    got_codes, got_params = g.leaf_codes()
    if codec == P.Codec.affine8:
        assert np.array_equal(got_codes, codes)
    else:
        unpacked = np.stack([got_codes & 15, got_codes >> 4], axis=-1).reshape(len(got_codes), 512)
        assert np.array_equal(unpacked, codes)
    assert np.array_equal(bits(got_params), bits(params))
    d = sc.dims
    c = all_coords((-1, -1, -1), (d[0] + 1, d[1] + 1, d[2] + 1))
    assert np.array_equal(bits(g.read_voxels(c)), bits(ref.open(deq).read_voxels(c)))
    # quantisation error bound: |v - decode(code(v))| <= scale/2 (+1 ulp)
    err = np.abs(g.read_voxels(c[:50000]).astype(np.float64) - ref.open(svdb).read_voxels(c[:50000]))
    assert err.max() <= params[:, 1].max() * 0.5 + 1e-6


def test_unorm8_rejects_non_byte_values(gpu):
    sc = S.scaled("C3", 32)
    _, svdb, _ = scene_svdb(sc)
    with pytest.raises(P.Error) as e:
        P.DeviceGrid(svdb, P.Codec.unorm8)
    assert e.value.code == P.Errc.size_mismatch
    assert P.DeviceGrid(svdb, P.Codec.auto8).codec == P.Codec.affine8


def test_sample_kats(gpu, ref):
    # test_sample.cpp:28-57
    g = P.DeviceGrid(ref.build_ops((16, 16, 16), 0.0, [(0, (5, 6, 7), 0.8125)]), P.Codec.f32)
    assert g.sample([[5.0, 6.0, 7.0]], 0)[0] == np.float32(0.8125)
    assert g.sample([[5.0, 6.0, 7.0]], 1)[0] == np.float32(0.8125)
    g = P.DeviceGrid(ref.build_ops((16, 16, 16), 0.0, [(0, (4, 4, 4), 0.0), (0, (5, 4, 4), 1.0)]), P.Codec.f32)
    assert g.sample([[4.5, 4.0, 4.0]], 1)[0] == np.float32(0.5)
    g = P.DeviceGrid(ref.build_ops((16, 16, 16), 0.375, [(0, (1, 1, 1), 5.0)]), P.Codec.f32)
    assert g.sample([[1e7, -1e7, 42.0], [1e30, 1e30, 1e30]], 1).tolist() == [0.375, 0.375]
    assert g.sample([[-1e18, 0.0, 0.0]], 0)[0] == np.float32(0.375)


@pytest.mark.parametrize("codec", [P.Codec.f32, P.Codec.auto8])
def test_sample_random_positions_bit_exact(gpu, ref, codec):
    # test_sample.cpp:59-73 domain (positions spill 6 voxels outside), 1e5 points + far outliers
    sc = S.scaled("C2", 4) if codec == P.Codec.auto8 else S.scaled("C3", 16)
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb, codec)
    rr = np.random.default_rng(500)
    d = np.array(sc.dims, np.float64)
    p = rr.uniform(0, 1, size=(100000, 3)) * (d + 12) - 6
    p = np.concatenate([p, [[1e30, 1e30, 1e30], [-1e18, 3, 4], [1e9 + 0.5, 2, 2], [np.nextafter(8.0, 0), 7.999, 15.0]]])
    rg = ref.open(svdb)
    for mode in (0, 1):
        assert np.array_equal(bits(g.sample(p, mode)), bits(rg.sample(p, mode)))
    assert np.array_equal(g.gradient(p[:20000]), rg.gradient(p[:20000]))


def test_macrocells_exact(gpu, ref, orc):
    # test_macrocell.cpp: ranges over closed 33^3 boxes + majorants (incl. KAT 1.6)
    sc = S.scaled("C2", 4)
    _, svdb, _ = scene_svdb(sc, quality=0.6)
    g = P.DeviceGrid(svdb, P.Codec.auto8)
    tf = sc.tf
    cells, cmin, cmax, maj, empty = g.macrocells(tf)
    rc = ref.open(svdb).macrocells(tf)
    assert cells == rc[0]
    for a, b in zip((cmin, cmax, maj), rc[1:4]):
        assert np.array_equal(bits(a), bits(b))
    assert np.array_equal(empty, rc[4])
    kat = P.DeviceGrid(ref.build_ops((32, 32, 32), 0.0, [(0, (1, 1, 1), 1.0)]), P.Codec.f32)
    tf2 = P.TransferFunction(0.0, 1.0, [[0, 0, 0, 0.1], [0, 0, 0, 0.8], [0, 0, 0, 0.3]], 2.0)
    _, _, _, m, e = kat.macrocells(tf2)
    assert m[0] == np.float32(1.6) and e[0] == 0


def test_svdb_errors_map_to_errc(gpu, ref):
    # test_io.cpp:71-134 corruption classes -> Errc
    svdb = bytearray(ref.build_ops((16, 16, 16), 0.0, [(0, (1, 2, 3), 1.0)]))
    bad = bytearray(svdb); bad[0:4] = b"XVDB"
    with pytest.raises(P.Error) as e:
        P.DeviceGrid(bytes(bad))
    assert e.value.code == P.Errc.bad_magic
    bad = bytearray(svdb); bad[4] = 3  # (2 is the quantised container, test_gpu_quantised.py)
    with pytest.raises(P.Error) as e:
        P.DeviceGrid(bytes(bad))
    assert e.value.code == P.Errc.version_mismatch
    with pytest.raises(P.Error) as e:
        P.DeviceGrid(bytes(svdb[:-1]))
    assert e.value.code == P.Errc.corrupt_index
    bad = bytearray(svdb)  # first lower slot payload of the upper -> out of range child
    nr = int(np.frombuffer(bytes(svdb[60:68]), np.uint64)[0])
    up = 72 + 16 * nr
    child = up + 16 + 4 * 32768
    slot = next(s for s in range(32768) if (bad[child + s // 8] >> (s % 8)) & 1)
    bad[up + 16 + 4 * slot: up + 20 + 4 * slot] = (999).to_bytes(4, "little")
    with pytest.raises(P.Error) as e:
        P.DeviceGrid(bytes(bad))
    assert e.value.code == P.Errc.corrupt_index


@pytest.mark.parametrize("codec", [P.Codec.f32, P.Codec.unorm8, P.Codec.affine8, P.Codec.affine4])
def test_apron_stencils_bit_exact_at_leaf_faces(gpu, orc, ref, codec):
    """Positions whose 2x2x2 stencil straddles leaf faces/edges/corners, lower-node boundaries,
    tiles and the volume border: the apron-backed gather must equal the reference sampler on the
    (dequantised) grid bit for bit."""
    sc = S.scaled("C2", 2) if codec == P.Codec.unorm8 else S.scaled("C3", 8)
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb, codec)
    deq = svdb if codec in (P.Codec.f32, P.Codec.unorm8) else orc.quantize(svdb, int(codec))[0]
    rg = ref.open(deq)
    if codec != P.Codec.unorm8:
        # leaves next to lower-slot tiles, upper-slot tiles and background (apron regions that
        # come from constants rather than neighbour leaves)
        ops = mixed_tile_ops(7, 400) + [(2, (128, 0, 0), 2.5), (0, (127, 5, 5), 9.0), (0, (135, 7, 7), 4.0)]
        tsv = ref.build_ops((200, 72, 72), 0.25, ops)
        tdeq = tsv if codec == P.Codec.f32 else orc.quantize(tsv, int(codec))[0]
        gt, rt = P.DeviceGrid(tsv, codec), ref.open(tdeq)
        pt = np.random.default_rng(5).uniform(-2, 1, size=(80000, 3)) + \
            np.random.default_rng(6).integers(0, 9, size=(80000, 3)) * 8 + 7
        pt[:, 0] *= 2.7
        assert np.array_equal(bits(gt.sample(pt, 1)), bits(rt.sample(pt, 1)))
    rr = np.random.default_rng(11)
    n = 60000
    d = np.array(sc.dims)
    base = rr.integers(-1, d + 1, size=(n, 3))
    base[: n // 2] = (base[: n // 2] // 8) * 8 + 7          # x/y/z all at a leaf's last voxel
    base[n // 2: 3 * n // 4, 0] = (base[n // 2: 3 * n // 4, 0] // 128) * 128 + 127  # lower-node faces
    p = base + rr.uniform(0, 1, size=(n, 3))
    assert np.array_equal(bits(g.sample(p, 1)), bits(rg.sample(p, 1)))
