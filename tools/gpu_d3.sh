#!/bin/bash
O=gpurun_out/${1:-d3}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "exit=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
SPQ_SCOPE_LOG=$O/c5_scopes.txt timeout 900 python tools/run_config.py C5 - 1 > $O/C5.log 2>&1
gzip -f $O/c5_scopes.txt
