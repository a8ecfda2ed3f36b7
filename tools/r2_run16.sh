mkdir -p gpurun_out
for Q in 1e-2 1e-1 1 10; do
  FPI_JACOBI_QUAD=$Q timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-c5 --steps 3 > gpurun_out/bench_c4_q$Q.json 2> /dev/null
done
for Q in 1e-2 1; do
  FPI_JACOBI_QUAD=$Q timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_q$Q.json 2> /dev/null
done
FPI_JACOBI_QUAD=1 timeout 1800 python -m pytest tests/test_linalg_gpu.py tests/test_pipeline_gpu.py tests/test_svd_gpu.py tests/test_fullsize_gpu.py -q -x > gpurun_out/gpu_tests16.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests16.log
echo done
