#!/bin/bash
# C3 timings x3 + fast GPU tests
O=gpurun_out/${1:-x}; mkdir -p $O
for rep in 1 2 3; do SPQ_TIMINGS=1 timeout 300 python tools/run_config.py C3 - 3 > $O/c3_$rep.log 2>&1; done
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > $O/pytest.log 2>&1; echo "exit=$?" >> $O/pytest.log
