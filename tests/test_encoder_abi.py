"""CPU: the native host encoder (byte-identical SVDB vs the reference's compress + serialize),
the C-ABI surface (every declared symbol exported, loadable without a GPU, fails loudly — never
falls back — when no device is visible), scene/TF validation and error mapping."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import _native as N
from paper_2504_04564_b200 import scenes as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("kind,dims,vt", [("marschner_lobb", (64, 64, 64), 0), ("fbm_smoke", (96, 80, 70), 0),
                                          ("turbulence", (70, 64, 40), 1), ("sparse", (100, 90, 80), 1),
                                          ("sparse", (130, 9, 260), 1), ("fbm_smoke", (1, 1, 1), 0)])
@pytest.mark.parametrize("quality", [1.0, 0.5, 0.1, 0.0])
def test_encoder_byte_identical_to_reference(ref, kind, dims, vt, quality):
    v = P.synth(kind, dims, seed=3)
    for metric in (0, 1, 2):
        mine, rep = P.compress(v, P.CompressionParams(quality, P.Metric(metric)), voxel_type=P.VoxelType(vt))
        theirs, rrep = ref.compress(v, voxel_type=vt, quality=quality, metric=metric)
        assert mine == theirs
        assert rep.voxels_activated == rrep["voxels_activated"]
        assert rep.bricks_activated == rrep["bricks_activated"]
        assert rep.frozen_bytes == rrep["frozen_bytes"] == len(mine)
        assert rep.background == rrep["background"]


def test_encoder_handles_negative_zero_and_uniform_regions(ref):
    v = np.zeros((40, 48, 56), np.float32)
    v[:, :, :24] = -0.0           # normalised to +0 (volume.hpp:61-62)
    v[8:16, 8:16, 8:16] = 0.75    # uniform, fully active leaf -> lower tile
    v[0:33, 0:33, 32:56] = 0.25   # large uniform blocks
    v[5, 6, 7] = 2.0
    for q in (1.0, 0.3):
        mine, _ = P.compress(v, P.CompressionParams(q))
        theirs, _ = ref.compress(v, voxel_type=1, quality=q)
        assert mine == theirs


def test_encoder_errors_match_reference_errc():
    with pytest.raises(P.Error) as e:
        P.compress(np.zeros((4, 4, 4), np.float32), P.CompressionParams(1.5))
    assert e.value.code == P.Errc.invalid_quality
    bad = np.zeros((4, 4, 4), np.float32)
    bad[1, 2, 3] = np.nan
    with pytest.raises(P.Error) as e:
        P.compress(bad)
    assert e.value.code == P.Errc.non_finite_voxel


def test_transfer_function_validation_mirrors_reference():
    # transfer.hpp:23-35
    for args in [(1.0, 1.0, [[0, 0, 0, 0]] * 2), (0.0, 1.0, [[0, 0, 0, 0]]), (0.0, 1.0, [[0, 0, 0, 1.5]] * 2)]:
        with pytest.raises(P.Error) as e:
            P.TransferFunction(*args)
        assert e.value.code == P.Errc.size_mismatch
    with pytest.raises(P.Error):
        P.TransferFunction(0.0, 1.0, [[0, 0, 0, 0]] * 2, density_scale=0.0)


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "svdbgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*(?:int|int64_t|void|const char\*)\s+(svdbgpu_\w+)\s*\(", src, flags=re.M))


def test_library_exports_every_declared_symbol():
    L = N.lib()
    declared = _declared_functions()
    assert declared == set(N.SIGNATURES), declared ^ set(N.SIGNATURES)
    for name in declared:
        assert hasattr(L, name), name
    assert L.svdbgpu_abi_version() == 1


def test_host_entry_points_need_no_gpu():
    assert P.tiles_for_rank(1920, 1080, 0, 1) == 120 * 68
    assert sum(P.tiles_for_rank(1920, 1080, r, 3) for r in range(3)) == 120 * 68
    assert P.tiles_for_rank(100, 100, 5, 3) == 0
    v = P.synth("turbulence", (8, 8, 8), 1)
    assert v.shape == (8, 8, 8) and 0.0 <= v.min() and v.max() <= 1.0


def test_nccl_loads_for_the_multi_device_render():
    # svdbgpu_render_multi resolves NCCL at first use (no link-time dependency); the library found here
    # is the one the NCCL gather would run on
    v = P.nccl_version()
    assert v >= 22700, v


def test_render_multi_validates_arguments_without_a_gpu():
    cam = P.Camera(width=16, height=16)
    tf = P.TransferFunction(0.0, 1.0, [[0, 0, 0, 0], [1, 1, 1, 1]])
    with pytest.raises(P.Error) as e:
        P.render_multi([], tf, cam, P.RenderSettings())
    assert e.value.status == P.api.E_INVALID_ARG


def test_device_calls_fail_loudly_without_gpu():
    if P.device_count() > 0:
        pytest.skip("a GPU is visible")
    svdb, _ = P.compress(P.synth("marschner_lobb", (16, 16, 16), 0), voxel_type=P.VoxelType.u8)
    with pytest.raises(P.Error) as e:
        P.DeviceGrid(svdb)
    assert e.value.code == P.api.E_NO_DEVICE


def test_corrupt_svdb_rejected_before_touching_the_device():
    with pytest.raises(P.Error) as e:
        P.DeviceGrid(b"XVDB" + bytes(100))
    assert e.value.code == P.Errc.bad_magic
    with pytest.raises(P.Error) as e:
        P.DeviceGrid(b"SVDB" + (3).to_bytes(4, "little") + bytes(100))
    assert e.value.code == P.Errc.version_mismatch
    # version 2 is the quantised container: its header is validated like v1's
    with pytest.raises(P.Error) as e:
        P.DeviceGrid(b"SVDB" + (2).to_bytes(4, "little") + bytes(100))
    assert e.value.code == P.Errc.corrupt_index


def test_scene_table_covers_baseline_configs():
    assert {"C1", "C2", "C3", "C4", "C5"} <= set(S.SCENES)
    c3 = S.SCENES["C3"]
    assert c3.dims == (1024, 1024, 1024) and (c3.width, c3.height) == (1920, 1080) and c3.settings.spp == 64
    assert S.SCENES["C4"].settings.mode == P.RenderMode.ratio
    assert S.SCENES["C1"].settings.mode == P.RenderMode.ea
