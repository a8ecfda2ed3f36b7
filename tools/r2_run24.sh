mkdir -p gpurun_out
FPI_DIST_BACKEND=gloo timeout 1200 python bench.py --gpus 8 --workload c4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c4_gloo8.json 2> gpurun_out/bench_c4_gloo8.err
echo exit=$? >> gpurun_out/bench_c4_gloo8.err
FPI_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 3 --workload c2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c2_gloo3.json 2> gpurun_out/bench_c2_gloo3.err
echo done
