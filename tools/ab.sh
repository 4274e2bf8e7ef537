#!/bin/bash
# usage: tools/ab.sh "<bench args>" variant1 variant2 ...   (runs on the GPU box)
args=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = "main" ]; then lib=""; else lib="paper_2504_04564_b200/csrc/build/variants/lib_$v.so"; fi
  SVDBGPU_LIB=${lib:-paper_2504_04564_b200/libsvdbgpu.so} timeout ${AB_TIMEOUT:-600} python bench.py --no-cpu-baseline --no-e2e --no-fp32 $args > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err || tail -3 gpurun_out/ab_$v.err
  python tools/summ.py gpurun_out/ab_$v.json
done
