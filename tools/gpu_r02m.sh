#!/bin/bash
# CPQR plan A/B on C3: per-level cpqr device time for forced variants / CTA sizes
O=gpurun_out/${1:-r02m}; mkdir -p $O
run() { tag=$1; shift; env "$@" timeout 300 python tools/run_config.py C3 - 4 > $O/c3_$tag.log 2>&1; }
run default SPQ_X=1
run v1 SPQ_CPQR_V1=1
for v in 0 3 4 6 7; do for nt in 128 256 512; do run var${v}_nt${nt} SPQ_CPQR_VAR=$v SPQ_CPQR_NTMIN=$nt; done; done
run var0_nt128_cl8 SPQ_CPQR_VAR=0 SPQ_CPQR_NTMIN=128 SPQ_CPQR_CLMAX=8
run var3_nt128_cl8 SPQ_CPQR_VAR=3 SPQ_CPQR_NTMIN=128 SPQ_CPQR_CLMAX=8
SPQ_CPQR_LOG=1 timeout 300 python tools/run_config.py C3 - 1 2>&1 >/dev/null | grep cpqr | awk '{print $5,$6,$7,$8}' | sort | uniq -c | sort -rn > $O/plans_default.txt
for f in $O/c3_*.log; do echo "$(basename $f) $(grep -E 'level (7|6|5|4|3|2):' $f | grep -oE 'cpqr=[0-9.]+' | tr '\n' ' ') $(grep -E '^factor' $f | tail -1)"; done > $O/summary.txt
