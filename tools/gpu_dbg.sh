mkdir -p gpurun_out/db
SPQ_SPEC_DEBUG=1 timeout 600 python tools/run_config.py C3 - 1 > gpurun_out/db/c3_spec.log 2>&1
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_kernels.py tests/test_gpu_batched.py -x -q -k "not slow" > gpurun_out/db/tests.log 2>&1; echo "exit=$?" >> gpurun_out/db/tests.log
timeout 600 python tools/run_config.py C3 - 3 > gpurun_out/db/c3.log 2>&1
timeout 600 python tools/run_config.py C4 - 2 > gpurun_out/db/c4.log 2>&1
