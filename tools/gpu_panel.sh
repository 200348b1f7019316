mkdir -p gpurun_out/pn
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_kernels.py tests/test_gpu_batched.py -x -q -k "not slow" > gpurun_out/pn/tests.log 2>&1; echo "exit=$?" >> gpurun_out/pn/tests.log
timeout 600 python tools/run_config.py C3 - 3 > gpurun_out/pn/c3.log 2>&1
CMD="python tools/run_config.py C3 - 1"
$CMD > gpurun_out/pn/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x --clock-control none -k regex:"panel_qr|chain_phase" --csv --log-file gpurun_out/pn/launches.csv $CMD > gpurun_out/pn/ncu.log 2>&1
echo "exit=$?" >> gpurun_out/pn/ncu.log
