mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "not c5" > gpurun_out/t17.log 2>&1; echo "exit=$?" >> gpurun_out/t17.log
SPQ_CPQR_CLUSTER=1 timeout 600 python -m pytest tests/test_gpu_factor.py -q -x --timeout 300 -k "not c4 and not c5" > gpurun_out/t17_cl.log 2>&1; echo "exit=$?" >> gpurun_out/t17_cl.log
timeout 300 python tools/run_config.py C3 - 3 > gpurun_out/c3_17.log 2>&1; echo "exit=$?" >> gpurun_out/c3_17.log
timeout 600 python tools/run_config.py C4 - 2 > gpurun_out/c4_17.log 2>&1; echo "exit=$?" >> gpurun_out/c4_17.log
