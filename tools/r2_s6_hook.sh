mkdir -p gpurun_out
for hk in 1 2 4; do for sh in 0 1; do
  echo "== hk=$hk short=$sh" >> gpurun_out/s6_hook.txt
  FPI_REORDER_HK=$hk FPI_REORDER_SHORT=$sh timeout 300 python tools/reorder_trace.py c4 4 2>&1 | grep -v generated >> gpurun_out/s6_hook.txt
  FPI_REORDER_HK=$hk FPI_REORDER_SHORT=$sh timeout 300 python tools/reorder_trace.py c5 4 2>&1 | grep -v generated >> gpurun_out/s6_hook.txt
done; done
FPI_REORDER_HK=1 FPI_REORDER_SHORT=1 timeout 600 python -m pytest tests/test_reorder_gpu.py -m gpu -q -x > gpurun_out/s6_hook_tests.log 2>&1
echo done
