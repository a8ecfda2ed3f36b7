mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/s6_margins_full.log 2>&1
grep -E "^\[sigma\]|rel|err|PASSED|FAILED" gpurun_out/s6_margins_full.log > gpurun_out/s6_margins.txt
rm -f gpurun_out/s6_margins_full.log.gz; gzip gpurun_out/s6_margins_full.log
echo done
