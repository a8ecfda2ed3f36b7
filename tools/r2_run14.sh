mkdir -p gpurun_out
for P in 1 2 3; do
  FPI_JACOBI_PASSES=$P timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-c5 --steps 3 > gpurun_out/bench_c4_p$P.json 2> gpurun_out/bench_c4_p$P.err
done
for P in 1 2; do
  FPI_JACOBI_PASSES=$P timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_p$P.json 2> gpurun_out/bench_c5_p$P.err
done
timeout 600 python tools/e2e_profile.py > gpurun_out/e2e_prof_c4.txt 2>&1
echo done
