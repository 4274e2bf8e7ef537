#!/bin/bash
# Copy a tools/measure_r2.sh run's artifacts from gpurun_out/ into profiles/ (summaries, lines,
# phases, launch list, bench lines, phase stats, tile balance). usage: tools/collect_profiles.sh [prefix]
P=${1:-r2}
cd "$(dirname "$0")/.."
for c in C3 C4; do
  python tools/ncu_summary.py gpurun_out/${P}_prof_$c.ncu-rep > profiles/${P}_ncu_k_trace_$c.txt
  python tools/ncu_lines.py gpurun_out/${P}_prof_$c.ncu-rep 400 > profiles/${P}_ncu_k_trace_${c}_lines.txt
  python tools/ncu_phases.py profiles/${P}_ncu_k_trace_${c}_lines.txt paper_2504_04564_b200/csrc/render.cu \
    paper_2504_04564_b200/csrc/device.cuh > profiles/${P}_ncu_k_trace_${c}_phases.txt
  sort -u gpurun_out/${P}_phase_stats_$c.txt > profiles/${P}_phase_stats_$c.txt
  grep '^{' gpurun_out/${P}_tile_balance_$c.log | tail -1 > profiles/${P}_tile_balance_$c.json
done
python tools/ncu_summary.py gpurun_out/${P}_prof_K2.ncu-rep > profiles/${P}_ncu_k_sample_K2.txt
python tools/launch_summary.py gpurun_out/${P}_launches_C3_bench_default.csv > profiles/${P}_launches_C3_summary.txt
cp gpurun_out/${P}_launches_C3_bench_default.csv profiles/
for c in C1 C2 C3 C3_4bit C4 C5; do cp gpurun_out/${P}_bench_$c.json profiles/${P}_bench_$c.json; done
cp gpurun_out/${P}_bench_K2.json profiles/${P}_bench_K2_sampler.json
cp gpurun_out/${P}_bench_reference.json profiles/${P}_bench_reference_arm.json
