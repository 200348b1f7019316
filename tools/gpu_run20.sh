mkdir -p gpurun_out
timeout 2000 python tools/diag_levels.py C5 64 > gpurun_out/lev64m.log 2>&1; echo "exit=$?" >> gpurun_out/lev64m.log
