mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "not c5" > gpurun_out/t24.log 2>&1; echo "exit=$?" >> gpurun_out/t24.log
timeout 300 python tools/run_config.py C3 - 3 > gpurun_out/c3_24.log 2>&1
timeout 300 python tools/solve_timing.py C3 > gpurun_out/solve24.log 2>&1
timeout 600 python tools/run_config.py C4 - 2 > gpurun_out/c4_24.log 2>&1
