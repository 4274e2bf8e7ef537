#!/usr/bin/env python3
"""Aggregate an ncu_lines.py dump of k_trace into code categories (phase / function) by source-line
ranges of the render.cu snapshot that was profiled. usage: ncu_phases.py <lines.txt> <render.cu snapshot>"""
import collections
import re
import sys

lines_txt, snap = sys.argv[1], sys.argv[2]
src = open(snap).read().splitlines()


def find(pat, start=0):
    for i in range(start, len(src)):
        if re.search(pat, src[i]):
            return i + 1
    raise SystemExit(f"pattern not found: {pat}")


marks = [  # (category, first line) in file order; a category runs to the next mark
    ("tracer-helpers", find(r"struct Tracer")),
    ("scatter", find(r"void isotropic\(")),
    ("tracer-helpers", find(r"// trace_path \(render.hpp:160-187\)")),
    ("camera", find(r"Ray camera_ray\(const CamArgs")),
    ("other", find(r"__global__ void __launch_bounds__\(256\) k_render")),
    ("dda-init", find(r"struct SharedDda")),
    ("dda-next", find(r"bool next\(const int cells\[3\], int cell\[3\]")),
    ("setup", find(r"^template <int CODEC, int MODE, bool CHUNK")),
    ("finish/scatter", find(r"auto finish_path")),
    ("start", find(r"auto do_start")),
    ("advance", find(r"auto do_advance")),
    ("exact-step", find(r"auto do_exact_step")),
    ("accept/sample", find(r"auto accept")),
    ("schedule", find(r"^    for \(;;\) \{", find(r"auto do_sample"))),
    ("other", find(r"__global__ void k_camera_rays|__global__ void k_unpack")),
]
marks.sort(key=lambda m: m[1])


def cat_render(n):
    c = "other"
    for name, start in marks:
        if n >= start:
            c = name
    return c


dev = open(sys.argv[3]).read().splitlines() if len(sys.argv) > 3 else []


def dfind(pat):
    for i, t in enumerate(dev):
        if re.search(pat, t):
            return i + 1
    return 10 ** 9


dmarks = sorted([("dev-layout", 1), ("gather", dfind(r"struct Accessor")), ("util", dfind(r"double dclamp\(")),
                 ("tf", dfind(r"double tf_normalized")), ("log", dfind(r"double step_log")),
                 ("rng", dfind(r"^__device__ __forceinline__ uint64_t mix64")), ("dda-dev", dfind(r"^struct Ray"))],
                key=lambda m: m[1])


def cat(f, n):
    if f == "render.cu":
        return cat_render(n)
    if f == "device.cuh" and dev:
        c = "device.cuh"
        for name, start in dmarks:
            if n >= start:
                c = name
        return c
    return f


rows = []
for l in open(lines_txt):
    m = re.match(r"(\S+)\s*:(\d+)\s+stall\s+([\d.]+)% inst\s+([\d.]+)% lanes\s+([\d.]+)", l)
    if m:
        rows.append((m.group(1), int(m.group(2)), float(m.group(3)), float(m.group(4)), float(m.group(5))))
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for f, n, st, ins, ln in rows:
    c = cat(f, n)
    agg[c][0] += st
    agg[c][1] += ins
    agg[c][2] += ins * ln
tot = sum(v[2] for v in agg.values())
print(f"{'category':18s} stall%  warp-inst%  lanes  thread-inst%")
for c, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{c:18s} {v[0]:6.2f}  {v[1]:9.2f}  {v[2] / max(v[1], 1e-9):5.1f}  {100 * v[2] / tot:9.2f}")
