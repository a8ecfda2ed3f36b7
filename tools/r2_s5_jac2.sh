mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_linalg_gpu.py tests/test_svd_gpu.py -m gpu -q -x -rf > gpurun_out/s5_jac_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/s5_jac_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-c5 > gpurun_out/s5_jac_c4.json 2> gpurun_out/s5_jac_c4.err
timeout 900 python bench.py --workload c5 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s5_jac_c5.json 2> gpurun_out/s5_jac_c5.err
timeout 900 python tools/jacobi_tune.py "" "FPI_JACOBI_CHUNKS=3,3" "FPI_JACOBI_CHUNKS=2,3" "FPI_JACOBI_CHUNKS=4,2" "FPI_JACOBI_CHUNKS=3,2" "FPI_JACOBI_CHUNKS=2,2" "FPI_JACOBI_CHUNKS=4,4" "FPI_JACOBI_CHUNKS=6,4" > gpurun_out/s5_jtune_c4.txt 2>&1
timeout 1200 python tools/jacobi_tune.py --workload=c5 "" "FPI_JACOBI_CHUNKS=3,8" "FPI_JACOBI_CHUNKS=2,8" "FPI_JACOBI_CHUNKS=4,4" "FPI_JACOBI_CHUNKS=3,4" "FPI_JACOBI_CHUNKS=2,4" "FPI_JACOBI_CHUNKS=4,6" "FPI_JACOBI_CHUNKS=6,8" "FPI_JACOBI_CHUNKS=2,2" > gpurun_out/s5_jtune_c5.txt 2>&1
echo done
