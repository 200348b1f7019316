#!/bin/bash
# round-2 first pass: GPU parity (incl. slow full configs), then the bench
O=gpurun_out/r02a; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -rA > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
