mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_linalg_gpu.py -q -x > gpurun_out/gpu_tests12a.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests12a.log
timeout 600 python tools/gemm_bench.py > gpurun_out/gemm_tma.txt 2>&1
FPI_GEMM_NO_TMA=1 timeout 600 python tools/gemm_bench.py gram_BtB_c4 gram_Yt_c4 gram_YtY_c5 YtU_c5 Gram_NT_c4 Z_L_NT_c4 > gpurun_out/gemm_notma.txt 2>&1
echo done
