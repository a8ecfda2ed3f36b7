mkdir -p gpurun_out
timeout 600 python tools/gap_trace.py c4 15 > gpurun_out/gaps_c4.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-c5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests22.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests22.log
echo done
