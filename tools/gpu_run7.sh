mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 280 > gpurun_out/t7.log 2>&1; echo "exit=$?" >> gpurun_out/t7.log
timeout 300 python tools/run_config.py C3 - 4 > gpurun_out/c3_7.log 2>&1; echo "exit=$?" >> gpurun_out/c3_7.log
