"""Synthetic BASELINE volumes: the product's svdbgpu_synth and the oracle's C restatement
(oracle/synth_oracle.c, what the reference arm of bench.py uses so it never loads libsvdbgpu.so)
are bit-identical, and the sparse C4 field hits its specified 35% +- 1% non-background leaf blocks
 with the per-size calibration, counted on the SVDB the reference's compress builds."""
import numpy as np
import pytest

import paper_2504_04564_b200 as P


@pytest.mark.parametrize("kind,dims,seed", [
    ("marschner_lobb", (64, 64, 64), 0), ("marschner_lobb", (33, 20, 17), 0),
    ("fbm_smoke", (64, 64, 64), 2), ("fbm_smoke", (50, 37, 29), 9),
    ("turbulence", (64, 64, 64), 3), ("turbulence", (41, 66, 23), 5),
    ("sparse", (64, 64, 64), 4), ("sparse", (128, 96, 72), 4), ("sparse", (200, 200, 200), 7)])
def test_product_and_oracle_synth_bit_identical(orc, kind, dims, seed):
    a = P.synth(kind, dims, seed, threads=4)
    b = orc.synth(kind, dims, seed, threads=3)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("n", [128, 256, 512])
def test_sparse_field_leaf_fraction_is_35_percent(orc, n):
    # the same per-size calibration the 2048^3 C4 volume uses (tools/calibrate_sparse.py)
    vol = orc.synth("sparse", (n, n, n), 4)
    blocks = vol.reshape(n // 8, 8, n // 8, 8, n // 8, 8)
    nonbg = (blocks != 0.0).any(axis=(1, 3, 5))
    frac = float(nonbg.mean())
    print(f"{n}^3: {100 * frac:.2f}% non-background leaf blocks, threshold {orc.sparse_threshold(n)}")
    assert abs(frac - 0.35) <= 0.01
    # the encoder keeps exactly those blocks as leaves (uniform all-1.0 blocks become tiles)
    svdb, rep = P.compress(vol, P.CompressionParams(1.0), voxel_type=P.VoxelType.f32)
    n_leaf = int(np.frombuffer(svdb[52:60], np.uint64)[0])
    uniform = ((blocks == 1.0).all(axis=(1, 3, 5))).sum()
    assert n_leaf + uniform == nonbg.sum() + (0 if nonbg[0, 0, 0] else 1) + (0 if nonbg[-1, -1, -1] else 1)
    assert abs(n_leaf / nonbg.size - 0.35) <= 0.01
