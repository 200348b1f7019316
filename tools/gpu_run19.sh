mkdir -p gpurun_out
timeout 900 python tools/diag_levels.py C5 48 > gpurun_out/lev48m.log 2>&1
timeout 1500 python tools/diag_levels.py C5 64 > gpurun_out/lev64m.log 2>&1
