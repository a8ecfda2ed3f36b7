mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_reorder_gpu.py tests/test_partition_gpu.py -q -x > gpurun_out/gpu_tests17a.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests17a.log
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x -k "reorder or partition" > gpurun_out/gpu_tests17b.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests17b.log
timeout 600 python tools/reorder_trace.py c4 3 > gpurun_out/reorder_prof_c4.txt 2>&1
echo done
