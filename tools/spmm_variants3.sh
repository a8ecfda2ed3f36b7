#!/bin/bash
# SpMM short-row path: slices per warp (FPI_SPMM_NSL) x unroll, benchmarked with tools/spmm_bench.py.
set -e
cd "$(dirname "$0")/../paper_2011_04235_b200/csrc"
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for u in 8 16; do
  $NV -DFPI_SPMM_UNROLL=$u -c spmm.cu -o build/spmm.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libfastpi_b200.so build/*.o
  for nsl in 1 2 4; do
    echo "== UNROLL $u NSL $nsl"
    (cd ../.. && FPI_SPMM_NSL=$nsl python tools/spmm_bench.py colblock_MX_k1000 A_X_k500 2>&1 | grep -v Warn | grep -v sparse_csr)
  done
done
touch spmm.cu && make -s
