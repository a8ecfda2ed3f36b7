mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_svd_gpu.py -m gpu -q -rf -s -k "ill_conditioned" > gpurun_out/s5_illcond_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/s5_illcond_tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_jacobi --launch-skip 5 -c 1 -o gpurun_out/s5_jacobi_c5_full -f python tools/run_once.py --workload c5 > gpurun_out/s5_ncu_jacobi_c5.log 2>&1
echo done
