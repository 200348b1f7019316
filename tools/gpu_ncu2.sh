mkdir -p gpurun_out/nc2
CMD="python tools/run_config.py C3 - 1"
$CMD > gpurun_out/nc2/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_qr_reg -s 150 -c 2 -o gpurun_out/nc2/panel $CMD > gpurun_out/nc2/ncu_panel.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_wave -s 300 -c 2 -o gpurun_out/nc2/chain $CMD > gpurun_out/nc2/ncu_chain.log 2>&1
echo "exit=$?" >> gpurun_out/nc2/ncu_chain.log
