mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "not c5" > gpurun_out/t26.log 2>&1; echo "exit=$?" >> gpurun_out/t26.log
timeout 300 python tools/solve_timing.py C3 > gpurun_out/solve26.log 2>&1
timeout 600 python tools/solve_timing.py C4 >> gpurun_out/solve26.log 2>&1
