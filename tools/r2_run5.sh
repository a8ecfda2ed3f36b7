mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_sharded_gpu.py tests/test_bench_gpu.py -q -x -rf --durations=10 > gpurun_out/gpu_tests5.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests5.log
echo done
