#!/bin/bash
# All BASELINE configs through bench.py on one GPU (runs on the GPU box): profiles/<round>_bench_<cfg>.json
round=${1:-r2}
mkdir -p gpurun_out
for cfg in C3 C3_4bit C5 C2 C4 C1; do
  extra=""
  [ "$cfg" = "C1" ] && extra="--no-fp32"
  timeout 1500 python bench.py --config $cfg --steps 5 --warmup 3 $extra > gpurun_out/${round}_bench_$cfg.json 2> gpurun_out/${round}_bench_$cfg.err
  echo "$cfg rc=$?"; python tools/summ.py gpurun_out/${round}_bench_$cfg.json
done
