mkdir -p gpurun_out
python tools/run_config.py C3 - 1 > gpurun_out/c3_22plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cpqr_cluster -s 10 -c 1 -o gpurun_out/prof_ccpqr python tools/run_config.py C3 - 1 > gpurun_out/ncu22.log 2>&1
echo "exit=$?" >> gpurun_out/ncu22.log
