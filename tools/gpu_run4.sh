mkdir -p gpurun_out
timeout 300 python tools/fp64_peak.py > gpurun_out/peak.log 2>&1; echo "exit=$?" >> gpurun_out/peak.log
timeout 300 python tools/run_config.py C3 - 1 > gpurun_out/c3_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/run_config.py C3 - 1 > gpurun_out/ncu_c3.log 2>&1; echo "exit=$?" >> gpurun_out/ncu_c3.log
