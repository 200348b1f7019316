mkdir -p gpurun_out/nc3
CMD="python tools/run_config.py C3 - 1"
$CMD > gpurun_out/nc3/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_qr_reg -s 150 -c 1 -o gpurun_out/nc3/panel $CMD > gpurun_out/nc3/ncu_panel.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cpqr_reg -s 40 -c 1 -o gpurun_out/nc3/cpqr $CMD > gpurun_out/nc3/ncu_cpqr.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_phaseA -s 500 -c 2 -o gpurun_out/nc3/chainA $CMD > gpurun_out/nc3/ncu_chain.log 2>&1
echo "exit=$?" >> gpurun_out/nc3/ncu_chain.log
