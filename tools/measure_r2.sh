#!/bin/bash
# Measurement set (tools/measure_r2.sh [prefix], default r2) (runs on the GPU box; results under gpurun_out/, summaries copied to profiles/)
P=${1:-r2}
mkdir -p gpurun_out
bash tools/bench_all.sh $P > gpurun_out/${P}_bench_all.log 2>&1; cat gpurun_out/${P}_bench_all.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${P}_bench_reference.json 2> gpurun_out/${P}_bench_reference.err; echo "reference rc=$?"
timeout 600 python bench.py --mode sample --steps 5 --warmup 2 > gpurun_out/${P}_bench_K2.json 2> gpurun_out/${P}_bench_K2.err; echo "K2 rc=$?"
for c in C3 C4; do bash tools/ab.sh "--steps 1 --warmup 1 --config $c" stats > /dev/null 2>&1; grep phase-stats gpurun_out/ab_stats.err > gpurun_out/${P}_phase_stats_$c.txt; done
for c in C3 C4; do timeout 900 python tools/tile_balance.py $c > gpurun_out/${P}_tile_balance_$c.log 2>&1; done
bash tools/prof.sh ${P}_prof_C3 > /dev/null 2>&1; echo "prof C3 rc=$?"
bash tools/prof.sh ${P}_prof_C4 --config C4 > /dev/null 2>&1; echo "prof C4 rc=$?"
[ "${HDDA_PROF:-0}" = 1 ] && bash tools/prof.sh ${P}_prof_C4_hdda --config C4 --hdda > /dev/null 2>&1; echo "prof C4 hdda rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sample -c 1 -o gpurun_out/${P}_prof_K2 python bench.py --mode sample --steps 1 --warmup 0 > gpurun_out/${P}_prof_K2.log 2>&1; echo "prof K2 rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${P}_launches_C3_bench_default.csv python bench.py --steps 2 --warmup 1 > gpurun_out/${P}_launches.log 2>&1; echo "launches rc=$?"
