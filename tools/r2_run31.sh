mkdir -p gpurun_out
python tools/gemm_bench.py XtZ_c4_odd XtZ_c4_even WZ_c4_odd G_c4_odd > gpurun_out/gemm31.txt 2>&1
for sp in 1 2 4 8 16; do echo "splits=$sp" >> gpurun_out/gemm31.txt; FPI_GEMM_SPLITS=$sp python tools/gemm_bench.py XtZ_c4_odd XtZ_c4_even >> gpurun_out/gemm31.txt 2>&1; done
FPI_GEMM_NO_TMA=1 python tools/gemm_bench.py XtZ_c4_even >> gpurun_out/gemm31.txt 2>&1
