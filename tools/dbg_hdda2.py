"""Debug: first differing pixels of the HDDA multi-bounce case (GPU vs oracle), then per-visit traces."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import scenes as S
from oracle.oracle import Oracle
from helpers import scene_svdb
sc = S.scaled("C4", 8, spp=1, image_factor=16)
_, svdb, _ = scene_svdb(sc)
g = P.DeviceGrid(svdb, P.Codec.f32)
og = Oracle().open(svdb)
cam = sc.camera()
for spp in (1,):
    st = P.RenderSettings(spp=spp, seed=7, max_bounces=64, rr_start_bounce=3, hdda=1)
    img = P.render(g, sc.tf, cam, st).pixels
    want, _, _ = og.render(sc.tf, cam, st)
    bad = np.argwhere(np.any(img.view(np.uint32) != want.view(np.uint32), axis=-1))
    print("spp", spp, "bad", len(bad), "of", img.shape[0] * img.shape[1], "first", bad[:8].tolist())
