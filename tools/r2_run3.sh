mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_pipeline_gpu.py tests/test_cli.py tests/test_fullsize_gpu.py -q -x > gpurun_out/gpu_tests3.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests3.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
FPI_GRAM_ROUTE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_c4_gram.json 2> gpurun_out/bench_c4_gram.err
timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
FPI_GRAM_HEAVY=128 timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_h128.json 2> gpurun_out/bench_c5_h128.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
  python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_c5.log 2>&1
echo done
