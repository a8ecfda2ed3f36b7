# Session 6: odd-stride operand repack in the GEMM dispatcher, A/B at c4 and c5
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_linalg_gpu.py -m gpu -q -x -rf > gpurun_out/s6_rp_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/s6_rp_tests.log
timeout 1200 python -m pytest tests/test_pipeline_gpu.py -m gpu -q -x -rf >> gpurun_out/s6_rp_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/s6_rp_tests.log
for v in off on off on; do
  if [ $v = off ]; then export FPI_GEMM_NO_REPACK=1; else unset FPI_GEMM_NO_REPACK; fi
  timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --no-c5 >> gpurun_out/s6_rp_c4_$v.json 2>> gpurun_out/s6_rp_c4_$v.err
done
for v in off on; do
  if [ $v = off ]; then export FPI_GEMM_NO_REPACK=1; else unset FPI_GEMM_NO_REPACK; fi
  timeout 900 python bench.py --workload c5 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s6_rp_c5_$v.json 2> gpurun_out/s6_rp_c5_$v.err
done
unset FPI_GEMM_NO_REPACK
FPI_GEMM_LOG=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-c5 > /dev/null 2> gpurun_out/s6_gemm_log_c4.txt
echo done
