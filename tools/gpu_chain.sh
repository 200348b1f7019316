mkdir -p gpurun_out/ch
timeout 900 python -m pytest tests/test_gpu_factor.py -x -q -k "not slow" > gpurun_out/ch/tests.log 2>&1; echo "exit=$?" >> gpurun_out/ch/tests.log
timeout 600 python tools/solve_timing.py C3 > gpurun_out/ch/solve.json 2>&1
SPQ_CHAIN_NO_W=1 timeout 600 python tools/solve_timing.py C4 > gpurun_out/ch/solve_c4_noW.json 2>&1
timeout 600 python tools/solve_timing.py C4 > gpurun_out/ch/solve_c4.json 2>&1
