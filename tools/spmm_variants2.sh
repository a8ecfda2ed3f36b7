#!/bin/bash
# SpMM gather cache-operator variants (FPI_SPMM_LOAD) x unroll, benchmarked with tools/spmm_bench.py.
set -e
cd "$(dirname "$0")/../paper_2011_04235_b200/csrc"
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for cfg in "0 8" "1 8" "2 8" "2 4" "1 4"; do
  set -- $cfg
  $NV -DFPI_SPMM_LOAD=$1 -DFPI_SPMM_UNROLL=$2 -c spmm.cu -o build/spmm.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libfastpi_b200.so build/*.o
  echo "== LOAD UNROLL = $cfg"
  (cd ../.. && python tools/spmm_bench.py colblock_MX_k1000 colblock_MtB_k1000 A_X_k500 At_B_k500)
done
touch spmm.cu && make -s
