# shapes and times of every DMMA GEMM in one c4 and one c5 solve + apply (FPI_GEMM_LOG)
mkdir -p gpurun_out
for w in c4 c5; do
  FPI_GEMM_LOG=1 timeout 600 python tools/run_once.py --workload $w > gpurun_out/gemm_log_$w.txt 2>&1
done
