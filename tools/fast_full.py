"""Full-size FP32 / mixed-precision tracking vs the FP64 frame (matched streams): relative RMSE."""
import os, sys, time
sys.path.insert(0, '.')
from dataclasses import replace
import numpy as np
import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import scenes as S

for name in sys.argv[1:] or ["C4", "C3"]:
    sc = S.SCENES[name]
    vol = P.synth(sc.volume, sc.dims, sc.volume_seed, threads=0)
    svdb, _ = P.compress(vol, P.CompressionParams(1.0), voxel_type=sc.voxel_type, threads=0)
    del vol
    g = P.DeviceGrid(svdb, sc.codec)
    cam = sc.camera()
    a = P.render(g, sc.tf, cam, sc.settings).pixels.astype(np.float64)
    for prec in [int(x) for x in os.environ.get("PRECS", "1,2").split(",")]:
        b = P.render(g, sc.tf, cam, replace(sc.settings, precision=prec)).pixels.astype(np.float64)
        rmse = np.sqrt(((a - b) ** 2).sum() / (a ** 2).sum())
        print(f"{name} precision {prec}: rel RMSE vs fp64 {rmse:.3e}", flush=True)
