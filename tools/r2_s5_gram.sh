mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_pipeline_gpu.py -m gpu -q -x -rf -k "gram_route or h11 or c4" > gpurun_out/s5_gram_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/s5_gram_tests.log
FPI_GRAM_NO_SPLIT=1 timeout 900 python bench.py --workload c5 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s5_gram_c5_nosplit.json 2> gpurun_out/s5_gram_c5_nosplit.err
timeout 900 python bench.py --workload c5 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s5_gram_c5_split.json 2> gpurun_out/s5_gram_c5_split.err
FPI_TRACE=1 timeout 600 python tools/run_once.py --workload c5 > gpurun_out/s5_gram_c5_trace.txt 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py -m gpu -q -x -rf > gpurun_out/s5_gram_fullsize.log 2>&1; echo tests_exit=$? >> gpurun_out/s5_gram_fullsize.log
echo done
