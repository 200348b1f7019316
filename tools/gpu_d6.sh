#!/bin/bash
O=gpurun_out/${1:-d6}; mkdir -p $O
SPQ_SCOPE_LOG=$O/c3_scopes.txt timeout 300 python tools/c3_timeline.py C3 > $O/c3tl.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_batched.py -m gpu -x -q > $O/pytest.log 2>&1; echo "exit=$?" >> $O/pytest.log
