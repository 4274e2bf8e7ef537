#!/bin/bash
# usage: tools/fvariants.sh "name:-DFLAG=1 -DFLAG2=2" ...   builds render_fast.cu variants (here, no GPU)
cd "$(dirname "$0")/../paper_2504_04564_b200/csrc" || exit 1
mkdir -p build/variants
for v in "$@"; do
  n=${v%%:*}; f=${v#*:}
  /usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xptxas -v -Xcompiler -fPIC \
    -I../../include -I. --expt-relaxed-constexpr $f -c render_fast.cu -o build/variants/render_fast_$n.o 2> build/variants/f_$n.log || { cat build/variants/f_$n.log; exit 1; }
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o build/variants/lib_$n.so \
    build/grid.o build/capi.o build/host_encoder.o build/render.o build/variants/render_fast_$n.o -lpthread || exit 1
  echo "variant $n: $(grep -A3 'k_trace_fILi2ELi0ELi0Ed\|k_trace_fILi2ELi0Ed' build/variants/f_$n.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
done
