mkdir -p gpurun_out
timeout 300 python tools/solve_timing.py C3 > gpurun_out/solve25.log 2>&1
timeout 600 python tools/solve_timing.py C4 >> gpurun_out/solve25.log 2>&1
