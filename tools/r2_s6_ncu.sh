# Session-6 ncu --set full captures at HEAD (c4, the bench workload): one launch each of the lift GEMM,
# the persistent reorder, the largest SpMM and the n = 1000 eigensolve, inside the second solve
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on --profile-from-start off"
timeout 900 $N --kernel-name-base demangled -k 'regex:k_gemm<1, 1, 1>' --launch-skip 1 -c 1 -o gpurun_out/s6_gemm_lift_c4 -f python tools/run_once.py --workload c4 > gpurun_out/s6_ncu_gemm.log 2>&1
timeout 900 $N -k regex:k_reorder_persistent -c 1 -o gpurun_out/s6_reorder_c4 -f python tools/run_once.py --workload c4 > gpurun_out/s6_ncu_reorder.log 2>&1
timeout 900 $N -k regex:k_jacobi --launch-skip 2 -c 1 -o gpurun_out/s6_jacobi_c4 -f python tools/run_once.py --workload c4 > gpurun_out/s6_ncu_jacobi.log 2>&1
timeout 900 $N --kernel-name-base function -k 'regex:^k_spmm_multi$' -c 7 -o gpurun_out/s6_spmm_c4 -f python tools/run_once.py --workload c4 > gpurun_out/s6_ncu_spmm.log 2>&1
for f in s6_gemm_lift_c4 s6_reorder_c4 s6_jacobi_c4; do
  python tools/ncu_summary.py gpurun_out/$f.ncu-rep > gpurun_out/$f.json 2> gpurun_out/$f.err
done
ncu -i gpurun_out/s6_spmm_c4.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,launch__grid_size > gpurun_out/s6_spmm_c4.csv 2>&1
echo done
