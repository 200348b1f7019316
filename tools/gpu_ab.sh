#!/bin/bash
# A/B of a switch on C3 timings + fast GPU tests.  usage: gpu_ab.sh OUT "ENV=1"
O=gpurun_out/${1:-ab}; mkdir -p $O
SPQ_TIMINGS=1 timeout 300 python tools/run_config.py C3 - 3 > $O/c3.log 2>&1; echo "exit=$?" >> $O/c3.log
env $2 SPQ_TIMINGS=1 timeout 300 python tools/run_config.py C3 - 3 > $O/c3_b.log 2>&1; echo "exit=$?" >> $O/c3_b.log
SPQ_SCOPE_LOG=$O/scope.txt SPQ_TIMINGS=1 timeout 300 python tools/run_config.py C3 - 1 > $O/c3s.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > $O/pytest.log 2>&1; echo "exit=$?" >> $O/pytest.log
