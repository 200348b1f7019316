mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -k "not c5" > gpurun_out/t23.log 2>&1; echo "exit=$?" >> gpurun_out/t23.log
timeout 300 python tools/run_config.py C3 - 3 > gpurun_out/c3_23.log 2>&1
