#!/usr/bin/env python3
"""Top SASS instructions of an .ncu-rep by warp-stall samples (with the dominant stall reason)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
ie = h.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[si] or 0) for r in data)
print(f"total stall samples {tot:.0f}")
ranked = sorted(range(len(data)), key=lambda k: -float(data[k][si] or 0))[:n]
for k in ranked:
    r = data[k]
    s = float(r[si] or 0)
    top = max(stall_cols, key=lambda c: float(r[c] or 0))
    print(f"{k:5d} {s / tot * 100:5.2f}% {h[top][6:]:14s} exec {float(r[ie] or 0) / 1e6:7.1f}M  {r[src][:90]}")
