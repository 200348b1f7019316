mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "not c5" > gpurun_out/t16.log 2>&1; echo "exit=$?" >> gpurun_out/t16.log
timeout 300 python tools/run_config.py C3 - 3 > gpurun_out/c3_16.log 2>&1; echo "exit=$?" >> gpurun_out/c3_16.log
timeout 600 python tools/run_config.py C4 - 2 > gpurun_out/c4_16.log 2>&1; echo "exit=$?" >> gpurun_out/c4_16.log
