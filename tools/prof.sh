#!/bin/bash
# usage: tools/prof.sh <name> <bench args...>   (runs on the GPU box; plain run first, then ncu)
name=$1; shift
mkdir -p gpurun_out
P="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e $*"
$P > gpurun_out/${name}_plain.json 2> gpurun_out/${name}_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:k_trace\|k_render -c 1 -o gpurun_out/${name} $P > gpurun_out/${name}_ncu.log 2>&1
tail -2 gpurun_out/${name}_ncu.log
