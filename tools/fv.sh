for v in main acc smp both; do
  if [ $v = main ]; then L=paper_2504_04564_b200/libsvdbgpu.so; else L=paper_2504_04564_b200/csrc/build/fv/lib_$v.so; fi
  echo "== $v"
  SVDBGPU_LIB=$L PRECS=2 timeout 300 python tools/fast_full.py C4 2>&1 | grep RMSE
  SVDBGPU_LIB=$L timeout 200 python bench.py --precision mixed --no-fp32 --no-cpu-baseline --no-e2e > gpurun_out/fv_$v.json 2>/dev/null; python tools/summ.py gpurun_out/fv_$v.json | sed 's/| samples.*//'
  SVDBGPU_LIB=$L timeout 200 python bench.py --config C4 --precision mixed --no-fp32 --no-cpu-baseline --no-e2e > gpurun_out/fv4_$v.json 2>/dev/null; python tools/summ.py gpurun_out/fv4_$v.json | sed 's/| samples.*//'
done
