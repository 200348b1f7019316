#!/bin/bash
# C3 device idle gaps + host sampling profile + per-level wall times in one call.
O=gpurun_out/${1:-gaps}; mkdir -p $O
SPQ_SCOPE_LOG=$O/c3_scopes.txt timeout 300 python tools/c3_timeline.py C3 > $O/c3tl.log 2>&1; echo "exit=$?" >> $O/c3tl.log
python tools/timeline_gaps.py $O/c3_scopes.txt 25 > $O/gaps.txt 2>&1
SPQ_HOST_PROFILE=$O/hp.txt timeout 300 python tools/run_config.py C3 - 8 > $O/c3.log 2>&1; echo "exit=$?" >> $O/c3.log
