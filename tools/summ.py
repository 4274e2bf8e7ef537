#!/usr/bin/env python3
"""Print a one-line summary of bench.py JSON lines read from files or stdin."""
import json
import sys

for path in sys.argv[1:] or ["-"]:
    f = sys.stdin if path == "-" else open(path)
    for line in f:
        line = line.strip()
        if not line.startswith("{"):
            continue
        j = json.loads(line)
        rf = j.get("roofline", {})
        print(f"{path}: {j.get('value', 0):.1f} {j.get('unit')} | {j.get('mlookups_per_s', 0):.0f} Mlookups/s | "
              f"frac {rf.get('frac', 0):.4f} | ms/step {j.get('ms_per_step', 0):.1f} | "
              f"samples/path {j.get('samples_per_path', 0):.2f} | {j.get('config', {}).get('workload', '')}")
        if j.get("mixed_precision_tracking"):
            q = j["mixed_precision_tracking"]
            print(f"    mixed-precision tracking: {q['value']:.1f} Mpaths/s | frac {q['roofline_frac']:.4f} | "
                  f"rel RMSE vs fp64 {q['rel_rmse_vs_fp64']:.2e}")
