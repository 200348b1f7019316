#!/bin/bash
# recycled task vectors: timing + parity + bench
O=gpurun_out/${1:-r02w}; mkdir -p $O
timeout 300 python tools/run_config.py C3 - 8 > $O/c3.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
