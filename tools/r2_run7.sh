mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-c5 > gpurun_out/ncu_launch_c4.log 2>&1
echo done
