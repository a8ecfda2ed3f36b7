mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:k_gemm -c 1 -o gpurun_out/gemm_tma_sq -f python tools/gemm_bench.py square_4096 > gpurun_out/ncu_tma.log 2>&1
FPI_GEMM_NO_TMA=1 timeout 600 ncu --set full --clock-control none -k regex:k_gemm -c 1 -o gpurun_out/gemm_cpa_sq -f python tools/gemm_bench.py square_4096 > gpurun_out/ncu_cpa.log 2>&1
echo done
