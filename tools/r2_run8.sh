mkdir -p gpurun_out
# one --set full capture each: the largest DMMA GEMM of a c4 solve (the apply lift, 27th k_gemm of
# the timed solve) and the transposed SpMM T^T B (long-row segments)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm --launch-skip 53 -c 1 \
  -o gpurun_out/gemm_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-c5 > gpurun_out/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_segments --launch-skip 6 -c 1 \
  -o gpurun_out/spmm_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-c5 > gpurun_out/ncu_spmm.log 2>&1
echo done
