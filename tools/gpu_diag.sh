mkdir -p gpurun_out/dg
timeout 600 python tools/run_config.py C3 - 3 > gpurun_out/dg/c3.log 2>&1
timeout 600 python tools/run_config.py C4 - 2 > gpurun_out/dg/c4.log 2>&1
timeout 600 python tools/run_config.py C1 - 3 > gpurun_out/dg/c1.log 2>&1
