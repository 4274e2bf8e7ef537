#!/usr/bin/env python3
"""Per-source-line totals of an .ncu-rep (needs -lineinfo + --import-source on): warp-level
instructions executed, thread instructions, stall samples and the dominant stall reason.
usage: ncu_lines.py <rep> [top_n] [kernel-substring]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
kern = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
def num(v):
    try:
        return float(v)
    except (TypeError, ValueError):  # rows whose source text broke the CSV quoting
        return 0.0


agg = defaultdict(lambda: defaultdict(float))
src_of = {}
path = func = None
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        path = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        func = row[1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or (kern and kern not in (func or "")):
        continue
    if not row[0].isdigit():
        continue  # SASS rows under a source line (already aggregated into the line row)
    d = {k: (v if v not in ("-", "") else "0") for k, v in zip(hdr[4:], row[4:])}
    key = (path, int(row[0]))
    src_of[key] = row[1][:70]
    a = agg[key]
    a["inst"] += num(d.get("Instructions Executed"))
    a["thr"] += num(d.get("Thread Instructions Executed"))
    a["stall"] += num(d.get("Warp Stall Sampling (All Samples)"))
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            a[k] += num(v)
tot_i = sum(a["inst"] for a in agg.values())
tot_s = sum(a["stall"] for a in agg.values())
print(f"total warp inst {tot_i:.3e}  stall samples {tot_s:.0f}")
for key in sorted(agg, key=lambda k: -agg[k]["stall"])[:top]:
    a = agg[key]
    st = max((k for k in a if k.startswith("stall_")), key=lambda k: a[k], default="stall_-")
    lanes = a["thr"] / a["inst"] if a["inst"] else 0
    print(f"{key[0]:12s}:{key[1]:<5d} stall {a['stall'] / tot_s * 100:5.2f}% inst {a['inst'] / tot_i * 100:5.2f}% "
          f"lanes {lanes:5.1f} {st[6:]:10s} | {src_of[key]}")
