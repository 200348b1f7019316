mkdir -p gpurun_out
timeout 300 python tools/run_config.py C3 - 4 > gpurun_out/c3_6.log 2>&1; echo "exit=$?" >> gpurun_out/c3_6.log
