#!/usr/bin/env python3
"""Calibrate the sparse (C4) field's threshold per volume size: 35% of the 8^3 leaf blocks must hold
non-background voxels. Uses the oracle's exact per-block maxima of the pre-threshold
density d (oracle/synth_oracle.c, bit-identical to svdbgpu_synth); prints the 65th percentile.

  python tools/calibrate_sparse.py 256 512 1024 2048 [--seed 4]
"""
import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def block_max(n, seed, threads=0):
    from oracle.oracle import Oracle
    L = Oracle().lib
    L.so_sparse_block_max.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_void_p]
    dims = np.array([n, n, n], np.int32)
    nb = ((n + 7) // 8) ** 3
    out = np.empty(nb, np.float64)
    rc = L.so_sparse_block_max(dims.ctypes.data, seed, threads, out.ctypes.data)
    assert rc == 0
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sizes", type=int, nargs="+")
    ap.add_argument("--seed", type=int, default=4)
    a = ap.parse_args()
    for n in a.sizes:
        t0 = time.time()
        bm = block_max(n, a.seed)
        q = np.sort(bm)
        k = int(round(0.65 * len(q)))
        th = 0.5 * (q[k - 1] + q[k])
        th4 = round(th, 4)
        frac = float(np.mean(bm > th4))
        print(f"size {n}: threshold {th:.6f} -> {th4:.4f}: {100 * frac:.2f}% blocks above "
              f"({time.time() - t0:.1f} s)", flush=True)


if __name__ == "__main__":
    main()
