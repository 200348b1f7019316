#!/bin/bash
O=gpurun_out/${1:-b2x}; mkdir -p $O
for r in 1 2; do timeout 900 python bench.py --no-cpu-baseline > $O/bench$r.json 2> $O/bench$r.err; done
SPQ_TIMINGS=1 timeout 300 python tools/run_config.py C3 - 3 > $O/c3.log 2>&1
