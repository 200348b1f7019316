#!/bin/bash
O=gpurun_out/${1:-d5}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "exit=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
SPQ_HOST_PROFILE=$O/hp.txt timeout 300 python tools/run_config.py C3 - 8 > $O/c3hp.log 2>&1
