"""Streaming device encoder: the volume streamed through the B200 in 32-slice
z-slabs, five passes, no dense host array. Its SVDB must be byte-identical to the host encoder
(svdbgpu_compress, itself byte-identical to the reference's compress + serialize_frozen, pinned in
tests/test_encoder_abi.py) for the device-generated synthetic volumes and for host callback slabs."""
import numpy as np
import pytest

import paper_2504_04564_b200 as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,dims,seed", [
    ("sparse", (64, 64, 64), 4), ("sparse", (70, 45, 33), 4), ("sparse", (128, 96, 100), 9),
    ("turbulence", (64, 64, 64), 3), ("turbulence", (33, 70, 65), 5),
    ("fbm_smoke", (64, 64, 64), 2), ("fbm_smoke", (50, 40, 97), 6)])
@pytest.mark.parametrize("quality,metric", [(1.0, P.Metric.median), (0.5, P.Metric.median), (0.3, P.Metric.closest),
                                            (0.7, P.Metric.farthest)])
def test_device_synth_encoder_is_byte_identical(gpu, kind, dims, seed, quality, metric):
    vt = P.VoxelType.u8 if kind == "fbm_smoke" else P.VoxelType.f32
    want, wrep = P.compress(P.synth(kind, dims, seed), P.CompressionParams(quality, metric), voxel_type=vt)
    got, rep, sec = P.synth_compress(kind, dims, seed, P.CompressionParams(quality, metric))
    assert len(got) == len(want)
    assert bytes(got) == want
    assert rep == wrep


def test_callback_encoder_is_byte_identical_on_edge_volumes(gpu):
    r = np.random.default_rng(5)
    vol = r.random((45, 70, 33), dtype=np.float32)
    vol[:, :, :20] = 0.25                      # uniform region -> tiles
    vol[10:20, 10:40, 5:9] = -0.0              # negative zeros (from_data normalises them)
    vol[30:45, 60:70, :] = 0.0                 # background-valued bricks
    dims = (vol.shape[2], vol.shape[1], vol.shape[0])
    for q in (1.0, 0.4):
        want, wrep = P.compress(vol, P.CompressionParams(q))
        got, rep, _ = P.compress_stream(lambda z0, nz: vol[z0:z0 + nz], dims, P.CompressionParams(q))
        assert bytes(got) == want and rep == wrep


def test_callback_encoder_errors(gpu):
    vol = np.zeros((40, 8, 8), np.float32)
    vol[35, 3, 3] = np.nan
    with pytest.raises(P.Error) as e:
        P.compress_stream(lambda z0, nz: vol[z0:z0 + nz], (8, 8, 40))
    assert e.value.code == P.Errc.non_finite_voxel

    def boom(z0, nz):
        raise RuntimeError("disk went away")
    with pytest.raises(RuntimeError, match="disk went away"):
        P.compress_stream(boom, (8, 8, 8))
    with pytest.raises(P.Error) as e:
        P.synth_compress("sparse", (8, 8, 8), 0, P.CompressionParams(1.5))
    assert e.value.code == P.Errc.invalid_quality
    with pytest.raises(P.Error):
        P.synth_compress("marschner_lobb", (8, 8, 8))  # needs the host libm: host encoder only
