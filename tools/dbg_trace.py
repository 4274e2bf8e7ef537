"""Debug: per-visit trace of one (pixel, sample) on the oracle (SO_TRACE) for the HDDA 256^3 case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2504_04564_b200 as P
from paper_2504_04564_b200 import scenes as S
from oracle.oracle import Oracle
from helpers import scene_svdb
x, y, s = (int(v) for v in sys.argv[1].split(","))
imf = int(os.environ.get("DBG_IMF", "32"))
spp = int(os.environ.get("DBG_SPP", "4"))
sc = S.scaled("C4", 8, spp=spp, image_factor=imf)
_, svdb, _ = scene_svdb(sc)
st = P.RenderSettings(spp=spp, seed=7, max_bounces=64, rr_start_bounce=3, hdda=1)
os.environ["SO_TRACE"] = f"{x},{y},{s}"
img, _, _ = Oracle().open(svdb).render(sc.tf, sc.camera(), st, threads=1)
print("oracle pixel", img[y, x].tolist())
if len(sys.argv) > 2:
    g = P.DeviceGrid(svdb, P.Codec.f32)
    gi = P.render(g, sc.tf, sc.camera(), st)
    print("gpu pixel", gi.pixels[y, x].tolist())
