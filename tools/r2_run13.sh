mkdir -p gpurun_out
timeout 600 python tools/reorder_trace.py c4 3 > gpurun_out/reorder_prof_c4.txt 2>&1
timeout 600 python tools/e2e_profile.py > gpurun_out/e2e_prof_c4.txt 2>&1
echo done
