mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pipeline_gpu.py tests/test_sparse_api_gpu.py tests/test_estimators_gpu.py tests/test_evaluate_gpu.py -q -x > gpurun_out/gpu_tests30.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests30.log
timeout 600 python bench.py --no-cpu-baseline --no-c5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python tools/gap_trace.py c4 15 > gpurun_out/gap30.txt 2>&1
timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo done
