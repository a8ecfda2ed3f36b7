mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_reorder_gpu.py tests/test_partition_gpu.py -q -x > gpurun_out/gpu_tests15a.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests15a.log
timeout 600 python tools/reorder_trace.py c4 3 > gpurun_out/reorder_prof_c4.txt 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x -k "reorder or partition" > gpurun_out/gpu_tests15b.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests15b.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-c5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo done
