#!/bin/bash
O=gpurun_out/${1:-lev}; mkdir -p $O
SPQ_TIMINGS=1 timeout 300 python tools/run_config.py C3 - 3 > $O/c3.log 2>&1; echo "exit=$?" >> $O/c3.log
