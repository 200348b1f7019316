#!/bin/bash
# Every BASELINE config on the device path: C1/C3/C4/C5 factor + GMRES timings
# (family breakdown), config 2 batched kernels.
O=gpurun_out/${1:-cfg}; mkdir -p $O
timeout 300 python tools/config2.py > $O/c2.json 2> $O/c2.err
for c in C1 C3 C4; do
  SPQ_TIMINGS=1 timeout 600 python tools/run_config.py $c - 3 > $O/$c.log 2>&1
done
SPQ_TIMINGS=1 timeout 1200 python tools/run_config.py C5 - 1 > $O/C5.log 2>&1
echo done >> $O/C5.log
