#!/usr/bin/env python3
"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel launches, total /
mean ms and share of the command's GPU time. usage: launch_summary.py <launches.csv>"""
import collections
import csv
import io
import re
import sys

rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in csv.DictReader(io.StringIO("".join(rows))):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("(anonymous namespace)::", "")
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "nsecond")
    ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
    agg[name][0] += 1
    agg[name][1] += ns
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'mean ms':>9s} {'share':>7s}")
for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {n:8d} {ns / 1e6:10.2f} {ns / 1e6 / n:9.3f} {100 * ns / tot:6.1f}%")
