mkdir -p gpurun_out
timeout 900 python tools/apply_profile.py c4 10 > gpurun_out/s6_apply_c4.txt 2>&1
nvidia-smi topo -m > gpurun_out/s6_topo.txt 2>&1
lscpu | grep -i "numa\|socket\|model name\|^CPU(s)" >> gpurun_out/s6_topo.txt 2>&1
echo done
