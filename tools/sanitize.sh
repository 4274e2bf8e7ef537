#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_case.py (runs on the GPU box);
# summaries -> gpurun_out/sanitize_<tool>.txt
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.txt | tail -1)"
done
