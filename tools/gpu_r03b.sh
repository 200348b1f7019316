#!/bin/bash
# copy granularity A/B (elements per CTA)
O=gpurun_out/${1:-r03b}; mkdir -p $O
run() { tag=$1; shift; env "$@" timeout 300 python tools/run_config.py C3 - 5 > $O/c3_$tag.log 2>&1; }
run g2048 SPQ_COPY_GRAN=2048
run adaptive SPQ_X=1
run g4096 SPQ_COPY_GRAN=4096
run g8192 SPQ_COPY_GRAN=8192
run g2048b SPQ_COPY_GRAN=2048
run adaptiveb SPQ_X=1
for f in $O/c3_*.log; do echo "$(basename $f) $(grep -E 'level (10|9|8|7|6|5|4|3):' $f | grep -oE 'copy=[0-9.]+' | tr '\n' ' ') $(grep -E '^factor' $f | tail -3 | tr '\n' ' ')"; done > $O/summary.txt
