mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_pipeline_gpu.py -q -x -rf -k "deferred" > gpurun_out/s6_defer_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/s6_defer_tests.log
timeout 600 python tools/defer_ab.py c4 20 > gpurun_out/s6_defer_ab_c4.txt 2>&1
timeout 900 python tools/defer_ab.py c5 6 > gpurun_out/s6_defer_ab_c5.txt 2>&1
echo done
