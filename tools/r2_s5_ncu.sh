# Session-5 ncu --set full captures (source-level: read with tools/ncu_source_top.py / ncu_summary.py)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_jacobi --launch-skip 5 -c 1 -o gpurun_out/s5_jacobi_c5_full2 -f python tools/run_once.py --workload c5 > gpurun_out/s5_ncu_jacobi_c5_2.log 2>&1
# second solve of run_once: k_spmm_multi launches per c5 solve = 6 -> skip 6 + 5 = the T C2 lift (largest)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_multi --launch-skip 11 -c 1 -o gpurun_out/s5_spmm_c5_full -f python tools/run_once.py --workload c5 > gpurun_out/s5_ncu_spmm_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reorder_persistent --launch-skip 1 -c 1 -o gpurun_out/s5_reorder_c4_full -f python tools/run_once.py --workload c4 > gpurun_out/s5_ncu_reorder_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_emit --launch-skip 2 -c 1 -o gpurun_out/s5_emit_c5_full -f python tools/run_once.py --workload c5 > gpurun_out/s5_ncu_emit_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_rows --launch-skip 1 -c 1 -o gpurun_out/s5_gramrows_c5_full -f python tools/run_once.py --workload c5 > gpurun_out/s5_ncu_gramrows_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k 'regex:^k_gram_rows$' --launch-skip 1 -c 1 -o gpurun_out/s5_gramrows_c5_full -f python tools/run_once.py --workload c5 > gpurun_out/s5_ncu_gramrows_c5.log 2>&1
# GEMM launches of one c5 solve: 185; the second solve's big ones -- capture 3 of the longest by skipping into the column update
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k 'regex:^k_gemm$' --launch-skip 355 -c 14 -o gpurun_out/s5_gemm_c5_full -f python tools/run_once.py --workload c5 > gpurun_out/s5_ncu_gemm_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k 'regex:^k_spmm_multi$' --launch-skip 12 -c 2 -o gpurun_out/s5_spmm2_c5_full -f python tools/run_once.py --workload c5 > gpurun_out/s5_ncu_spmm2_c5.log 2>&1
echo done
