mkdir -p gpurun_out/dg2
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_kernels.py tests/test_gpu_batched.py -x -q -k "not slow" > gpurun_out/dg2/tests.log 2>&1; echo "exit=$?" >> gpurun_out/dg2/tests.log
timeout 900 python -m pytest tests/test_gpu_factor.py -x -q -k "c3_full or c4_full" > gpurun_out/dg2/tests_full.log 2>&1; echo "exit=$?" >> gpurun_out/dg2/tests_full.log
timeout 600 python tools/run_config.py C3 - 3 > gpurun_out/dg2/c3.log 2>&1
SPQ_SPARSIFY_PREFIX=1 timeout 600 python tools/run_config.py C3 - 3 > gpurun_out/dg2/c3_prefix.log 2>&1
timeout 600 python tools/run_config.py C4 - 2 > gpurun_out/dg2/c4.log 2>&1
timeout 300 python tools/config2.py > gpurun_out/dg2/config2.json 2>&1
