# Session-5 probe: GEMM shape logs (c4, c5) + smoke at HEAD
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/s5_smoke.log
for w in c4 c5; do
  FPI_GEMM_LOG=1 timeout 600 python tools/run_once.py --workload $w > gpurun_out/gemm_log_$w.txt 2>&1
done
echo done
