mkdir -p gpurun_out
timeout 300 python tools/kbench.py > gpurun_out/kbench.log 2>&1; echo "exit=$?" >> gpurun_out/kbench.log
CUDA_LAUNCH_BLOCKING=1 timeout 1500 python tools/run_config.py C5 - 1 > gpurun_out/c5_10.log 2>&1; echo "exit=$?" >> gpurun_out/c5_10.log
