# Session-6 evidence at HEAD: full GPU tests, smoke, default bench, reference arm, launch list, Amdahl
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/s6f_gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/s6f_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6f_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/s6f_smoke.log
timeout 1500 python bench.py > gpurun_out/s6f_bench.json 2> gpurun_out/s6f_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s6f_bench_ref.json 2> gpurun_out/s6f_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s6f_launches_c4.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-c5 > gpurun_out/s6f_ncu_launch.log 2>&1
timeout 900 python tools/shard_amdahl.py c4 3 > gpurun_out/s6f_amdahl_c4.json 2> /dev/null
timeout 1200 python tools/shard_amdahl.py c5 2 > gpurun_out/s6f_amdahl_c5.json 2> /dev/null
echo done
