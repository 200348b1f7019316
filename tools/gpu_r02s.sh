#!/bin/bash
# round-2 ncu --set full captures (one launch each, after a plain run): CPQR, panel QR, larft, DMMA GEMM, chain A/B
O=gpurun_out/${1:-r02s}; mkdir -p $O
CMD="python tools/run_config.py C3 - 1"
$CMD > $O/plain.log 2>&1 || exit 1
cap() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o $O/$3 $CMD > $O/ncu_$3.log 2>&1; echo "exit=$?" >> $O/ncu_$3.log; }
cap cpqr_reg 120 cpqr
cap panel_qr_reg 250 panel
cap larft_blk 120 larft
cap gemm_dmma2 40 gemm
cap chain_phaseA 30 chainA
cap chain_phaseB 30 chainB
cap copy_tasks 150 copy
for f in cpqr panel larft gemm chainA chainB copy; do python tools/ncu_summary.py $O/$f.ncu-rep > $O/$f.summary.txt 2>&1; done
