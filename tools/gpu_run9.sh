mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "not c5" > gpurun_out/t9.log 2>&1; echo "exit=$?" >> gpurun_out/t9.log
timeout 300 python tools/run_config.py C3 - 3 > gpurun_out/c3_9.log 2>&1; echo "exit=$?" >> gpurun_out/c3_9.log
timeout 600 python tools/run_config.py C4 - 2 > gpurun_out/c4_9.log 2>&1; echo "exit=$?" >> gpurun_out/c4_9.log
timeout 1200 python tools/run_config.py C5 - 1 > gpurun_out/c5_9.log 2>&1; echo "exit=$?" >> gpurun_out/c5_9.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/c5_9.log
