#!/bin/bash
# Memory-safety check of record (compute-sanitizer is closed on the GPU pool): the bounds-checked build
# (csrc/Makefile variants: checked:-DSVDB_CHECKED=1, device asserts on every indexed hot-path load and
# store) over every kernel family (tools/sanitize_case.py) and one full-size C3 frame.
mkdir -p gpurun_out
lib=paper_2504_04564_b200/csrc/build/variants/lib_checked.so
SVDBGPU_LIB=$lib timeout 900 python tools/sanitize_case.py > gpurun_out/checked_case.txt 2>&1; echo "case rc=$?"
SVDBGPU_LIB=$lib timeout 900 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-fp32 > gpurun_out/checked_c3.json 2> gpurun_out/checked_c3.err; echo "C3 full frame rc=$?"
grep -h "SVDB_ASSERT" gpurun_out/checked_case.txt gpurun_out/checked_c3.err | head -5
