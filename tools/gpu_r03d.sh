#!/bin/bash
# same-box A/B: allocator tracking, copy granularity (interleaved, per-call medians)
O=gpurun_out/${1:-r03d}; mkdir -p $O
for rep in 1 2; do
  SPQ_ALLOC_TRACK_ALL=1 python tools/stall_probe.py > $O/calls_tracked_$rep.txt 2>&1
  python tools/stall_probe.py > $O/calls_untracked_$rep.txt 2>&1
done
for f in $O/calls_*.txt; do echo "$(basename $f) $(head -1 $f | cut -c1-28) $(grep -E '# +(0|3|7|10|14|17) ' $f | awk '{printf "%s ", $NF}') $(tail -1 $f)"; done > $O/summary.txt
