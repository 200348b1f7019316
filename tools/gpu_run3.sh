mkdir -p gpurun_out
timeout 300 python tools/run_config.py C3 - 3 > gpurun_out/c3.log 2>&1; echo "exit=$?" >> gpurun_out/c3.log
timeout 300 python -m pytest tests/test_gpu_kernels.py -q --timeout 280 > gpurun_out/t3.log 2>&1; echo "exit=$?" >> gpurun_out/t3.log
