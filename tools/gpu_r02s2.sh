#!/bin/bash
# second ncu --set full pass: the three latency-bound kernels (skip counts inside one factorization)
O=gpurun_out/${1:-r02s}; mkdir -p $O
CMD="python tools/run_config.py C3 - 1"
$CMD > $O/plain2.log 2>&1 || exit 1
cap() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o $O/$3 $CMD > $O/ncu_$3.log 2>&1; echo "exit=$?" >> $O/ncu_$3.log; }
cap cpqr_reg 60 cpqr
cap panel_qr_reg 150 panel
cap larft_blk 60 larft
for f in cpqr panel larft; do python tools/ncu_summary.py $O/$f.ncu-rep > $O/$f.summary.txt 2>&1; python tools/ncu_lines.py $O/$f.ncu-rep > $O/$f.lines.txt 2>&1; done
for f in gemm chainA chainB copy; do [ -f $O/$f.ncu-rep ] && python tools/ncu_lines.py $O/$f.ncu-rep > $O/$f.lines.txt 2>&1; done
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
