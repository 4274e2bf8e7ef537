#!/usr/bin/env python3
"""Load balance of the interleaved 16x16 tile split measured on ONE GPU: for N
ranks, render each rank's tile set separately (independent renders, no collective) and report the
per-rank kernel times. max(rank time) bounds an N-GPU frame; mean/max is the balance efficiency.
This is evidence for the split, not a multi-GPU measurement."""
import json
import sys

sys.path.insert(0, ".")
import paper_2504_04564_b200 as P  # noqa: E402
from paper_2504_04564_b200 import scenes as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
sc = S.SCENES[name]
svdb, _, _ = P.synth_compress(sc.volume, sc.dims, sc.volume_seed)  # streaming device encoder
g = P.DeviceGrid(svdb, sc.codec)
cam = sc.camera()
P.render(g, sc.tf, cam, sc.settings)  # warm-up (majorants, caches)
P.render(g, sc.tf, cam, sc.settings, tile_rank=0, tile_nranks=2)  # warm-up of the split path's buffers
full = P.render(g, sc.tf, cam, sc.settings).stats["render_ms"]
out = {"config": name, "full_frame_ms": full, "splits": {}}
for n in (2, 4, 8):
    t = [P.render(g, sc.tf, cam, sc.settings, tile_rank=r, tile_nranks=n).stats["render_ms"] for r in range(n)]
    out["splits"][n] = {"rank_ms": t, "max_ms": max(t), "mean_ms": sum(t) / n,
                        "balance": (sum(t) / n) / max(t), "ideal_speedup_bound": full / max(t)}
    print(f"{name} N={n}: rank ms {[round(x, 1) for x in t]} balance {(sum(t) / n) / max(t):.3f} "
          f"full/max {full / max(t):.2f}", flush=True)
print(json.dumps(out))
