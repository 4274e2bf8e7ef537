"""Debug: HDDA GPU vs oracle on the sparse field (prints identical fractions)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import scenes as S
from oracle.oracle import Oracle
from helpers import image_parity, scene_svdb
orc = Oracle()
for factor, imf, codec in ((32, 32, P.Codec.f32), (8, 32, P.Codec.f32), (8, 32, P.Codec.affine8)):
    sc = S.scaled("C4", factor, spp=4, image_factor=imf)
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb, codec)
    deq = orc.quantize(svdb, int(codec))[0] if int(codec) else svdb
    og = orc.open(deq)
    cam = sc.camera()
    for hd in (0, 1):
        st = P.RenderSettings(spp=4, seed=7, max_bounces=64, rr_start_bounce=3, hdda=hd)
        img = P.render(g, sc.tf, cam, st)
        want, lk, _ = og.render(sc.tf, cam, st)
        same, rmse = image_parity(img.pixels, want)
        bad = np.argwhere(np.any(img.pixels.view(np.uint32) != want.view(np.uint32), axis=-1))
        print(f"{sc.dims[0]}^3 {codec.name} hdda={hd}: identical {same:.4f} rmse {rmse:.2e} lookups gpu {img.stats['lookups']} oracle {lk} first bad {bad[:3].tolist()}")
