mkdir -p gpurun_out
for L in paper_2504_04564_b200/libsvdbgpu.so paper_2504_04564_b200/csrc/build/variants/lib_noreb.so; do
  echo "== $L" >> gpurun_out/exp.log
  SVDBGPU_LIB=$L PRECS=1 timeout 400 python tools/fast_full.py C4 C3 >> gpurun_out/exp.log 2>&1
  SVDBGPU_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-fp32 --precision fp32 --steps 3 --warmup 3 > gpurun_out/exp_b.json 2>/dev/null; python tools/summ.py gpurun_out/exp_b.json >> gpurun_out/exp.log 2>&1
done
