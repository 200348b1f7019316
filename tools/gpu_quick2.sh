#!/bin/bash
O=gpurun_out/${1:-q}; mkdir -p $O
SPQ_TIMINGS=1 timeout 300 python tools/run_config.py C3 - 3 > $O/c3.log 2>&1; echo "exit=$?" >> $O/c3.log
for r in 128 512 1024; do SPQ_PANEL_ROWS=$r SPQ_TIMINGS=1 timeout 300 python tools/run_config.py C3 - 3 > $O/c3_rows$r.log 2>&1; done
SPQ_HOST_PROFILE=$O/hp.txt timeout 300 python tools/run_config.py C3 - 8 > $O/c3hp.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > $O/pytest.log 2>&1; echo "exit=$?" >> $O/pytest.log
