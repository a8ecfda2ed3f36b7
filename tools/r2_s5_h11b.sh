mkdir -p gpurun_out
FPI_GRAM_H11_GEMM=1 timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s5_h11b_c5_gemm.json 2> gpurun_out/s5_h11b_c5_gemm.err
timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s5_h11b_c5_id.json 2> gpurun_out/s5_h11b_c5_id.err
timeout 1200 python -m pytest tests/test_pipeline_gpu.py -m gpu -q -x -rf -k "gram_route or h11" > gpurun_out/s5_h11b_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/s5_h11b_tests.log
echo done
