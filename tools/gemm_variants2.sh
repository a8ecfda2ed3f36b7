#!/bin/bash
# DMMA GEMM k-tile depth (FPI_GEMM_CFG_BK) x stages x CTAs per SM, benchmarked with tools/gemm_bench.py.
set -e
cd "$(dirname "$0")/../paper_2011_04235_b200/csrc"
for cfg in "16 3 3" "32 2 3" "32 3 2" "32 4 2"; do
  set -- $cfg
  D="-DFPI_GEMM_CFG_BK=$1 -DFPI_GEMM_CFG_STAGES=$2 -DFPI_GEMM_CFG_CTAS=$3"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $D -c gemm.cu -o build/gemm.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libfastpi_b200.so build/*.o
  echo "== BK STAGES CTAS = $cfg"
  (cd ../.. && python tools/gemm_bench.py gram_BtB_c4 U_eq_B_Mx_c4 Z_VtT_WT_c4 gram_Yt_c4 square_4096 gram_YtY_c5 U_eq_Y_X_c5 2>&1 | sed 's/  (cuBLAS.*//')
done
