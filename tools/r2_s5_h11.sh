mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_pipeline_gpu.py -m gpu -q -x -rf -k "gram_route or h11" > gpurun_out/s5_h11_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/s5_h11_tests.log
FPI_GRAM_H11_GEMM=1 timeout 600 python tools/run_once.py --workload c5 --reps 3 > gpurun_out/s5_h11_c5_gemm.txt 2>&1
timeout 600 python tools/run_once.py --workload c5 --reps 3 > gpurun_out/s5_h11_c5_id.txt 2>&1
FPI_TRACE=1 timeout 600 python tools/run_once.py --workload c5 > gpurun_out/s5_h11_c5_trace.txt 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py -m gpu -q -x -rf > gpurun_out/s5_h11_fullsize.log 2>&1; echo tests_exit=$? >> gpurun_out/s5_h11_fullsize.log
echo done
