mkdir -p gpurun_out
(free -g; nproc) > gpurun_out/s4_host.txt
timeout 1500 python -m pytest tests/test_fullsize_gpu.py -q -x -rf -s --durations=10 > gpurun_out/s4_fullsize.log 2>&1; echo exit=$? >> gpurun_out/s4_fullsize.log
