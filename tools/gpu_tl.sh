#!/bin/bash
O=gpurun_out/${1:-tl}; mkdir -p $O
timeout 300 python tools/run_config.py C3 - 1 > $O/c3.log 2>&1
SPQ_SCOPE_LOG=$O/scope.txt SPQ_TIMINGS=1 timeout 300 python tools/run_config.py C3 - 1 > $O/c3s.log 2>&1; echo "exit=$?" >> $O/c3s.log
