mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/t8.log 2>&1; echo "exit=$?" >> gpurun_out/t8.log
timeout 300 python tools/run_config.py C3 - 3 > gpurun_out/c3_8.log 2>&1; echo "exit=$?" >> gpurun_out/c3_8.log
timeout 300 python tools/config2.py > gpurun_out/config2.log 2>&1; echo "exit=$?" >> gpurun_out/config2.log
timeout 600 python tools/run_config.py C4 - 2 > gpurun_out/c4.log 2>&1; echo "exit=$?" >> gpurun_out/c4.log
