"""Small renders of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
k_leaf_encode / k_build_apron / k_build_dir (grid build), k_cell_ranges + k_majorants (macrocells),
k_camera_rays + k_trace (pathtrace / ratio, chunked and whole-pixel, HDDA), k_reduce, k_render (EA /
ISO), k_sample, the streaming encoder kernels and k_unpack, on a 64^3 sparse grid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import scenes as S

sc = S.scaled("C4", 32, spp=4, image_factor=120)          # 64^3 sparse, 32x18
svdb, _, _ = P.synth_compress(sc.volume, sc.dims, sc.volume_seed)   # streaming encoder kernels
cam = sc.camera()
for codec in (P.Codec.affine8, P.Codec.f32):
    g = P.DeviceGrid(svdb, codec)
    g.macrocells(sc.tf)
    for st in (P.RenderSettings(spp=16, seed=1), P.RenderSettings(spp=2, seed=1, mode=P.RenderMode.ratio),
               P.RenderSettings(spp=16, seed=1, mode=P.RenderMode.ratio, hdda=1, majorant_cell=8),
               P.RenderSettings(spp=1, mode=P.RenderMode.ea), P.RenderSettings(spp=1, mode=P.RenderMode.iso),
               P.RenderSettings(spp=16, seed=1, precision=2)):
        img = P.render(g, sc.tf, cam, st)
        assert np.isfinite(img.pixels).all()
    img = P.render(g, sc.tf, cam, P.RenderSettings(spp=8), tile_rank=1, tile_nranks=3)
    xs = np.random.default_rng(0).random((1000, 3)) * 70 - 3
    g.sample(xs, 1)
    g.read_voxels(np.zeros((4, 3), np.int32))
print("sanitize case done")
