#!/bin/bash
# DMMA GEMM at two CTAs per SM: parity, C3 and C4 bench
O=gpurun_out/${1:-r03h}; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err; echo "exit=$?" >> $O/bench_C4.err
