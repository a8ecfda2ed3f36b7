# Session 5: dense core of T (sparse_core.cu): parity tests + c4 / c5 A-B against the plain SpMM
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_pipeline_gpu.py -m gpu -q -x -rf -k "sparse_core or stagewise_parity_c4 or test_stagewise_parity" --durations=5 > gpurun_out/s5_core_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/s5_core_tests.log
for v in 0 1; do
  if [ $v = 0 ]; then export FPI_SPMM_CORE=0; else unset FPI_SPMM_CORE; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-c5 > gpurun_out/s5_core_c4_$v.json 2> gpurun_out/s5_core_c4_$v.err
  FPI_TRACE=1 timeout 600 python tools/run_once.py --workload c4 > gpurun_out/s5_core_trace_c4_$v.txt 2>&1
  timeout 600 python tools/run_once.py --workload c5 --reps 3 > gpurun_out/s5_core_c5_$v.txt 2>&1
done
echo done
