#!/bin/bash
O=gpurun_out/${1:-chk}; mkdir -p $O
SPQ_TIMINGS=1 timeout 300 python tools/run_config.py C3 - 3 > $O/c3.log 2>&1; echo "exit=$?" >> $O/c3.log
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "exit=$?" >> $O/pytest.log
