#!/bin/bash
# usage: tools/prof_lib.sh <name> <variant> <bench args...>
name=$1; v=$2; shift 2
mkdir -p gpurun_out
lib=paper_2504_04564_b200/csrc/build/variants/lib_$v.so
[ "$v" = "main" ] && lib=paper_2504_04564_b200/libsvdbgpu.so
P="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e $*"
SVDBGPU_LIB=$lib $P > gpurun_out/${name}_plain.json 2> gpurun_out/${name}_plain.err && \
SVDBGPU_LIB=$lib ncu --set full --clock-control none --import-source on -k regex:k_trace\|k_render -c 1 -o gpurun_out/${name} $P > gpurun_out/${name}_ncu.log 2>&1
tail -1 gpurun_out/${name}_ncu.log
