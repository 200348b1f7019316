mkdir -p gpurun_out
timeout 2000 python tools/diag_levels.py C5 64 > gpurun_out/lev64m.log 2>&1; echo "exit=$?" >> gpurun_out/lev64m.log
timeout 600 python -m pytest tests/test_gpu_factor.py tests/test_gpu_kernels.py tests/test_gpu_batched.py -q --timeout 300 -k "not c4 and not c5" > gpurun_out/t21.log 2>&1; echo "exit=$?" >> gpurun_out/t21.log
SPQ_CPQR_CLUSTER=1 timeout 600 python -m pytest tests/test_gpu_factor.py -q -x --timeout 300 -k "not c4 and not c5" > gpurun_out/t21_cl.log 2>&1; echo "exit=$?" >> gpurun_out/t21_cl.log
timeout 300 python tools/run_config.py C3 - 3 > gpurun_out/c3_21.log 2>&1
