mkdir -p gpurun_out
timeout 900 python tools/defer_ab.py c4 12 > gpurun_out/s6_e2e_ab_c4.txt 2>&1
timeout 1200 python tools/defer_ab.py c5 5 > gpurun_out/s6_e2e_ab_c5.txt 2>&1
echo done
