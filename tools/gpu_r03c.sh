#!/bin/bash
# allocator: untracked block memory; copy granularity: per-call times, parity (incl. slow), bench
O=gpurun_out/${1:-r03c}; mkdir -p $O
python tools/stall_probe.py > $O/calls.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
