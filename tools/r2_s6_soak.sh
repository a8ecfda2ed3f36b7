mkdir -p gpurun_out
for i in 1 2; do
  timeout 2400 python -m pytest tests -m gpu -q -x -rf -p no:cacheprovider > gpurun_out/s6_soak_$i.log 2>&1; echo tests_exit=$? >> gpurun_out/s6_soak_$i.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6_soak_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/s6_soak_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s6_soak_bench.json 2> gpurun_out/s6_soak_bench.err; echo bench_exit=$? >> gpurun_out/s6_soak_smoke.log
echo done
