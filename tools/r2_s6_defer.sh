mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_pipeline_gpu.py tests/test_capi.py -q -x -rf -k "deferred or c_abi or capi or symbol" > gpurun_out/s6_defer_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/s6_defer_tests.log
for v in off on off on; do
  if [ $v = off ]; then export FPI_NO_DEFERRED_UPLOAD=1; else unset FPI_NO_DEFERRED_UPLOAD; fi
  timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-c5 >> gpurun_out/s6_defer_c4_$v.json 2>> gpurun_out/s6_defer_c4_$v.err
done
for v in off on; do
  if [ $v = off ]; then export FPI_NO_DEFERRED_UPLOAD=1; else unset FPI_NO_DEFERRED_UPLOAD; fi
  timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s6_defer_c5_$v.json 2> gpurun_out/s6_defer_c5_$v.err
done
echo done
