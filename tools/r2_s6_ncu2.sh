mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on --profile-from-start off"
timeout 1200 $N --kernel-name-base function -k 'regex:^k_gemm$' -c 40 -o gpurun_out/s6_gemm_c4 -f python tools/run_once.py --workload c4 > gpurun_out/s6_ncu_gemm.log 2>&1
ncu -i gpurun_out/s6_gemm_c4.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread > gpurun_out/s6_gemm_c4.csv 2>&1
echo done
