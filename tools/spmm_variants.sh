#!/bin/bash
# Build the CSR SpMM with several (unroll, min CTAs/SM) settings and benchmark each (tools/spmm_bench.py).
# A file tools/ubench/spmm_old.cu, when present, is benchmarked first as the "before" variant.
set -e
cd "$(dirname "$0")/../paper_2011_04235_b200/csrc"
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
if [ -f ../../tools/ubench/spmm_old.cu ]; then
  cp ../../tools/ubench/spmm_old.cu spmm_old_tmp.cu
  $NV -c spmm_old_tmp.cu -o build/spmm.o && rm spmm_old_tmp.cu
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libfastpi_b200.so build/*.o
  echo "== old"
  (cd ../.. && python tools/spmm_bench.py "$@")
fi
for cfg in "8 3" "8 2" "4 4" "6 4" "4 3"; do
  set -- $cfg
  $NV -DFPI_SPMM_UNROLL=$1 -DFPI_SPMM_MINB=$2 -c spmm.cu -o build/spmm.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libfastpi_b200.so build/*.o
  echo "== UNROLL MINB = $cfg"
  (cd ../.. && python tools/spmm_bench.py)
done
touch spmm.cu && make -s
