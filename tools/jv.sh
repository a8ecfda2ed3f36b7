timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/jv.log
FPI_JACOBI_PROFILE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep "jacobi" | head -8 >> gpurun_out/jv.log
timeout 300 python tools/bench_ab.py >> gpurun_out/jv.log 2>&1
