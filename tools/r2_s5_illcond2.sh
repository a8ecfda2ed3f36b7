mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_svd_gpu.py -m gpu -q -rf -s > gpurun_out/s5_illcond2_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/s5_illcond2_tests.log
timeout 900 python -m pytest tests/test_pipeline_gpu.py -m gpu -q -x -rf -k "not c4" > gpurun_out/s5_illcond2_pipe.log 2>&1; echo tests_exit=$? >> gpurun_out/s5_illcond2_pipe.log
echo done
