"""Shared test data builders (mirroring the reference tests' own constructions)."""
from __future__ import annotations

import numpy as np

import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import scenes as S


class SplitMix:
    """svdb::Rng(seed) (rng.hpp:35-60) in Python, so randomized cases mirror the reference's."""

    M = (1 << 64) - 1

    def __init__(self, seed: int):
        self.state = self.mix64(seed)

    @staticmethod
    def mix64(x: int) -> int:
        M = SplitMix.M
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)

    def next_u64(self) -> int:
        M = self.M
        self.state = (self.state + 0x9E3779B97F4A7C15) & M
        x = self.state
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53


def random_voxel_ops(seed=2024, n=5000, dim=64):
    """Freeze.RandomizedOracleEquivalence (test_tree.cpp:160-182) op stream."""
    r = SplitMix(seed)
    ops = []
    for _ in range(n):
        c = (int(r.uniform() * dim), int(r.uniform() * dim), int(r.uniform() * dim))
        v = float(np.float32(r.uniform() * 10.0))
        ops.append((0, c, v))
    return ops, r


def mixed_tile_ops(seed=7, n=400):
    """Freeze.MixedTileAndVoxelOpsMatchReference (test_tree.cpp:184-217) op stream."""
    r = SplitMix(seed)
    ops = []
    for _ in range(n):
        pick = r.uniform()
        if pick < 0.2:
            o = (8 * int(r.uniform() * 8), 8 * int(r.uniform() * 8), 8 * int(r.uniform() * 8))
            ops.append((1, o, float(np.float32(r.uniform() * 5.0))))
        else:
            c = (int(r.uniform() * 64), int(r.uniform() * 64), int(r.uniform() * 64))
            ops.append((0, c, float(np.float32(r.uniform() * 5.0))))
    return ops


def all_coords(lo, hi):
    g = np.mgrid[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]].reshape(3, -1)
    return np.ascontiguousarray(np.stack([g[2], g[1], g[0]], axis=1).astype(np.int32))


def scene_svdb(scene: S.Scene, quality=1.0):
    vol = P.synth(scene.volume, scene.dims, scene.volume_seed)
    data, rep = P.compress(vol, P.CompressionParams(quality), voxel_type=scene.voxel_type)
    return vol, data, rep


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


# Bit-identical pixel fraction required of FP64 GPU frames against the reference / oracle: the
# measured value is 1.0 on every scene (CUDA's log / sincos may differ from glibc in the last ulp,
# which could flip one decision of a path; the build with SVDB_GLIBC_LOG=1 removes the log case).
MIN_IDENTICAL = 0.999


def image_parity(got: np.ndarray, want: np.ndarray):
    """-> (fraction of bit-identical pixels, relative RMSE = rms(got-want)/rms(want))."""
    same = np.all(bits(got) == bits(want), axis=-1).mean()
    d = got.astype(np.float64) - want.astype(np.float64)
    denom = np.sqrt(np.mean(want.astype(np.float64) ** 2)) or 1.0
    return float(same), float(np.sqrt(np.mean(d * d)) / denom)
