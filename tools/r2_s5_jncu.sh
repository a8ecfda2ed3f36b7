mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_jacobi --launch-skip 5 -c 1 -o gpurun_out/s5_jacobi_c5_full2 -f python tools/run_once.py --workload c5 > gpurun_out/s5_ncu_jacobi_c5_2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_jacobi --launch-skip 5 -c 1 -o gpurun_out/s5_jacobi_c4_full2 -f python tools/run_once.py --workload c4 > gpurun_out/s5_ncu_jacobi_c4_2.log 2>&1
echo done
