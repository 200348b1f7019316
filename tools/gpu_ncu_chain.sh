#!/bin/bash
# ncu --set full of the solve-chain kernels inside the solve phase (after the plain run exits 0)
O=gpurun_out/${1:-ncuchain}; mkdir -p $O
CMD="python tools/solve_timing.py C3"
$CMD > $O/plain.log 2>&1 || exit 1
cap() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c $3 -o $O/$4 $CMD > $O/ncu_$4.log 2>&1; echo "exit=$?" >> $O/ncu_$4.log; }
# first application of solve_w: waves 13..37 are the single-op root separators
cap chain_phaseA 75 3 chainA
cap chain_phaseB 40 2 chainB
for f in chainA chainB; do python tools/ncu_summary.py $O/$f.ncu-rep > $O/$f.summary.txt 2>&1; python tools/ncu_lines.py $O/$f.ncu-rep > $O/$f.lines.txt 2>&1; done
cat $O/chainA.summary.txt $O/chainB.summary.txt
