mkdir -p gpurun_out/pf2
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_kernels.py tests/test_gpu_batched.py -x -q -k "not slow" > gpurun_out/pf2/tests.log 2>&1; echo "exit=$?" >> gpurun_out/pf2/tests.log
SPQ_HOST_PROFILE=gpurun_out/pf2/c3.prof timeout 600 python tools/run_config.py C3 - 4 > gpurun_out/pf2/c3.log 2>&1
timeout 600 python tools/run_config.py C4 - 2 > gpurun_out/pf2/c4.log 2>&1
timeout 600 python tools/solve_timing.py C3 > gpurun_out/pf2/solve.json 2>&1
