# Session-4 re-entry check at HEAD: full GPU tests, smoke, default bench line.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -rf --durations=15 > gpurun_out/s4_gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/s4_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/s4_smoke.log
timeout 1500 python bench.py > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err
echo done
