mkdir -p gpurun_out
python tools/run_config.py C3 - 1 > gpurun_out/c3_18plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x --clock-control none -k regex:cpqr --csv --log-file gpurun_out/launches_cpqr.csv python tools/run_config.py C3 - 1 > gpurun_out/ncu18.log 2>&1
echo "exit=$?" >> gpurun_out/ncu18.log
