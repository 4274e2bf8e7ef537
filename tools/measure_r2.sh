#!/bin/bash
# Round-2 measurement set (runs on the GPU box; results under gpurun_out/, summaries copied to profiles/)
mkdir -p gpurun_out
bash tools/bench_all.sh r2 > gpurun_out/r2_bench_all.log 2>&1; cat gpurun_out/r2_bench_all.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err; echo "reference rc=$?"
timeout 600 python bench.py --mode sample --steps 5 --warmup 2 > gpurun_out/r2_bench_K2.json 2> gpurun_out/r2_bench_K2.err; echo "K2 rc=$?"
for c in C3 C4; do bash tools/ab.sh "--steps 1 --warmup 1 --config $c" stats > /dev/null 2>&1; grep phase-stats gpurun_out/ab_stats.err > gpurun_out/r2_phase_stats_$c.txt; done
for c in C3 C4; do timeout 900 python tools/tile_balance.py $c > gpurun_out/r2_tile_balance_$c.log 2>&1; done
bash tools/prof.sh r2_prof_C3 > /dev/null 2>&1; echo "prof C3 rc=$?"
bash tools/prof.sh r2_prof_C4 --config C4 > /dev/null 2>&1; echo "prof C4 rc=$?"
bash tools/prof.sh r2_prof_C4_hdda --config C4 --hdda > /dev/null 2>&1; echo "prof C4 hdda rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sample -c 1 -o gpurun_out/r2_prof_K2 python bench.py --mode sample --steps 1 --warmup 0 > gpurun_out/r2_prof_K2.log 2>&1; echo "prof K2 rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2_launches_C3_bench_default.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r2_launches.log 2>&1; echo "launches rc=$?"
