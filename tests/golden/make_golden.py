#!/usr/bin/env python3
"""Regenerate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libsvdbref.so, built
from /root/reference/proj/include by oracle/Makefile). Run here (where /root/reference exists):

    python tests/golden/make_golden.py

The fixtures pin the oracle and the GPU path on machines where the reference is absent. Inputs
are generated deterministically (the reference's own synth-style constructions, seeded), so the
script is the full provenance of every number stored.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle.oracle import Reference  # noqa: E402
from helpers import SplitMix, mixed_tile_ops, random_voxel_ops  # noqa: E402

import paper_2504_04564_b200 as P  # noqa: E402  (synth only: input generation)


def main():
    ref = Reference()
    out = {}
    # 1. randomized voxel grid (test_tree.cpp:160-182) + reads incl. out of bounds
    ops, r = random_voxel_ops(2024, 5000, 64)
    g1 = ref.build_ops((64, 64, 64), 0.5, ops)
    q = np.array([[int(r.uniform() * 80) - 8 for _ in range(3)] for _ in range(4000)], np.int32)
    out["voxels_svdb"] = np.frombuffer(g1, np.uint8)
    out["voxels_coords"] = q
    out["voxels_values"] = ref.open(g1).read_voxels(q)
    # 2. tiles grid (test_tree.cpp:184-217), pruned
    g2 = ref.build_ops((64, 64, 64), 0.0, mixed_tile_ops(7, 400), prune=True)
    out["tiles_svdb"] = np.frombuffer(g2, np.uint8)
    c = np.ascontiguousarray(np.stack(np.meshgrid(np.arange(-1, 65, 3), np.arange(-1, 65, 3),
                                                  np.arange(-1, 65, 3), indexing="ij"), -1).reshape(-1, 3)
                             .astype(np.int32))
    out["tiles_coords"] = c
    out["tiles_values"] = ref.open(g2).read_voxels(c)
    # 3. compressed Marschner-Lobb 32^3 from u8 (compress q=1 and q=0.5) + samples + render
    vol = P.synth("marschner_lobb", (32, 32, 32), 0)
    svdb, rep = ref.compress(vol, voxel_type=0, quality=1.0)
    svdb_half, _ = ref.compress(vol, voxel_type=0, quality=0.5)
    out["ml_volume"] = vol
    out["ml_svdb"] = np.frombuffer(svdb, np.uint8)
    out["ml_half_svdb_sha256"] = np.frombuffer(hashlib.sha256(svdb_half).digest(), np.uint8)
    rg = ref.open(svdb)
    rr = np.random.default_rng(7)
    pts = rr.uniform(-4, 36, size=(4000, 3))
    out["ml_points"] = pts
    out["ml_trilinear"] = rg.sample(pts, 1)
    out["ml_nearest"] = rg.sample(pts, 0)
    out["ml_gradient"] = rg.gradient(pts[:1000])
    tf = P.TransferFunction(0.0, 1.0, [[0, 0, 0, 0], [0.2, 0.8, 0.6, 0.3], [1.0, 0.3, 0.1, 0.9]], 0.5)
    out["tf_entries"] = tf.entries
    cells, cmin, cmax, maj, empty = rg.macrocells(tf)
    out["ml_cells"] = np.array(cells, np.int32)
    out["ml_cmin"], out["ml_cmax"], out["ml_maj"], out["ml_empty"] = cmin, cmax, maj, empty
    cam = P.Camera(position=(40.0, 35.0, -30.0), look_at=(15.5, 15.5, 15.5), width=32, height=24)
    out["cam"] = np.array([*cam.position, *cam.look_at, *cam.up, cam.fov_y_deg, cam.width, cam.height])
    st = P.RenderSettings(spp=4, max_bounces=64, rr_start_bounce=3, seed=11)
    out["pt_image"] = rg.render(tf, cam, st)
    sti = P.RenderSettings(spp=1, seed=3, mode=P.RenderMode.iso, iso_value=0.55, background_color=(0.1, 0.2, 0.3))
    out["iso_image"] = rg.render(tf, cam, sti)
    # 4. splitmix64 streams (rng.hpp:45-63)
    out["rng"] = np.stack([ref.rng_uniforms(s, px, py, k, 8) for (s, px, py, k) in
                           [(0, 0, 0, 0), (11, 5, 7, 3), (2 ** 63 + 5, -1, 4096, 63)]])
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"), {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
