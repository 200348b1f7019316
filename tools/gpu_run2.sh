mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -k "not slow" --timeout 240 > gpurun_out/t2.log 2>&1; echo "exit=$?" >> gpurun_out/t2.log
timeout 300 python tools/run_config.py C3 - 2 > gpurun_out/c3.log 2>&1; echo "exit=$?" >> gpurun_out/c3.log
timeout 300 python -m pytest tests -m "gpu and slow" -q --timeout 280 > gpurun_out/t2slow.log 2>&1; echo "exit=$?" >> gpurun_out/t2slow.log
