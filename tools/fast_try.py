import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, time
import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import scenes as S
from helpers import scene_svdb, image_parity
from dataclasses import replace
for name, f, fi, spp in [("C3",16,8,4),("C3",16,8,64),("C3",4,4,16),("C2",4,4,16),("C1",1,2,16),("C4",32,16,16)]:
    sc = S.scaled(name, f, spp=spp, image_factor=fi)
    _, svdb, _ = scene_svdb(sc)
    g = P.DeviceGrid(svdb, P.Codec.affine8 if name in ("C3","C4") else P.Codec.auto8)
    cam = sc.camera()
    st = replace(sc.settings, spp=spp)
    if name == "C1": st = replace(st, mode=P.RenderMode.pathtrace)
    a = P.render(g, sc.tf, cam, st).pixels
    b = P.render(g, sc.tf, cam, replace(st, precision=1)).pixels
    m = P.render(g, sc.tf, cam, replace(st, precision=2)).pixels
    c = P.render(g, sc.tf, cam, replace(st, seed=st.seed+1)).pixels
    same, rmse = image_parity(b, a)
    samem, rmsem = image_parity(m, a)
    _, rmse_noise = image_parity(c, a)
    print(f"{name} f{f} {cam.width}x{cam.height} spp{spp} {st.mode.name}: fp32 rmse {rmse:.2e} | mixed rmse {rmsem:.2e} | other-seed {rmse_noise:.2e}")
