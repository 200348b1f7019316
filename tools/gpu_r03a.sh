#!/bin/bash
# host threads in execute_wave, load without sync, merge flag OR: A/B + per-call times + parity + bench
O=gpurun_out/${1:-r03a}; mkdir -p $O
SPQ_HOST_THREADS=1 python tools/stall_probe.py > $O/calls_t1.txt 2>&1
python tools/stall_probe.py > $O/calls_t4.txt 2>&1
SPQ_HOST_THREADS=8 python tools/stall_probe.py > $O/calls_t8.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
