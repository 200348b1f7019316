#!/bin/bash
# quick loop: C3 timings + host profile + fast GPU tests
O=gpurun_out/${1:-q}; mkdir -p $O
SPQ_TIMINGS=1 timeout 300 python tools/run_config.py C3 - 3 > $O/c3.log 2>&1; echo "exit=$?" >> $O/c3.log
SPQ_HOST_PROFILE=$O/hp.txt timeout 300 python tools/run_config.py C3 - 8 > $O/c3hp.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > $O/pytest.log 2>&1; echo "exit=$?" >> $O/pytest.log
