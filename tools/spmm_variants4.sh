#!/bin/bash
# SpMM (two slices per warp): minimum resident CTAs per SM (FPI_SPMM_MINB), tools/spmm_bench.py.
set -e
cd "$(dirname "$0")/../paper_2011_04235_b200/csrc"
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for mb in 2 3 4; do
  $NV -DFPI_SPMM_MINB=$mb -c spmm.cu -o build/spmm.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libfastpi_b200.so build/*.o
  echo "== MINB $mb"
  (cd ../.. && python tools/spmm_bench.py colblock_MX_k1000 colblock_MtB_k1000 A_X_k500 At_B_k500 2>&1 | grep -v Warn | grep -v sparse_csr)
done
