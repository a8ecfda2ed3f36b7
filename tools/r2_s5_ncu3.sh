mkdir -p gpurun_out
# second solve of run_once: k_spmm_multi launches per c5 solve = 6 -> skip 6 + 5 = the T C2 lift (largest)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_multi --launch-skip 11 -c 1 -o gpurun_out/s5_spmm_c5_full -f python tools/run_once.py --workload c5 > gpurun_out/s5_ncu_spmm_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reorder_persistent --launch-skip 1 -c 1 -o gpurun_out/s5_reorder_c4_full -f python tools/run_once.py --workload c4 > gpurun_out/s5_ncu_reorder_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_emit --launch-skip 2 -c 1 -o gpurun_out/s5_emit_c5_full -f python tools/run_once.py --workload c5 > gpurun_out/s5_ncu_emit_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_rows --launch-skip 1 -c 1 -o gpurun_out/s5_gramrows_c5_full -f python tools/run_once.py --workload c5 > gpurun_out/s5_ncu_gramrows_c5.log 2>&1
echo done
