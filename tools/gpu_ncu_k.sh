#!/bin/bash
# ncu --set full of the two latency-bound kernels at C3 (one launch each)
O=gpurun_out/${1:-nk}; mkdir -p $O
CMD="python tools/run_config.py C3 - 1"
$CMD > $O/plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cpqr_reg -s 60 -c 1 -o $O/cpqr $CMD > $O/ncu_cpqr.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_qr_reg -s 200 -c 1 -o $O/panel $CMD > $O/ncu_panel.log 2>&1
echo done >> $O/ncu_panel.log
