#!/bin/bash
# Build the DMMA GEMM with several tile configurations and benchmark each (tools/gemm_bench.py).
set -e
cd "$(dirname "$0")/../paper_2011_04235_b200/csrc"
for cfg in "128 64 32 32 3 2" "64 64 32 32 3 3" "64 32 32 16 3 4" "64 32 32 16 3 5" "64 64 32 32 4 2" "128 128 64 32 3 1"; do
  set -- $cfg
  D="-DFPI_GEMM_CFG_BM=$1 -DFPI_GEMM_CFG_BN=$2 -DFPI_GEMM_CFG_WM=$3 -DFPI_GEMM_CFG_WN=$4 -DFPI_GEMM_CFG_STAGES=$5 -DFPI_GEMM_CFG_CTAS=$6"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $D -c gemm.cu -o build/gemm.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libfastpi_b200.so build/*.o
  echo "== BM BN WM WN STAGES CTAS = $cfg"
  (cd ../.. && python tools/gemm_bench.py gram_BtB_c4 U_eq_B_Mx_c4 Z_VtT_WT_c4 square_4096 gram_YtY_c5 U_eq_Y_X_c5 2>&1 | sed 's/  (cuBLAS.*//')
done
