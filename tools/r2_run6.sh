mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_sharded_gpu.py tests/test_bench_gpu.py -q -x -rf --durations=10 > gpurun_out/gpu_tests6.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests6.log
timeout 900 python tools/shard_amdahl.py c4 3 > gpurun_out/amdahl_c4.json 2> gpurun_out/amdahl_c4.err
timeout 1200 python tools/shard_amdahl.py c5 2 > gpurun_out/amdahl_c5.json 2> gpurun_out/amdahl_c5.err
echo done
