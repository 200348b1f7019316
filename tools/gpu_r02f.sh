#!/bin/bash
# round-2 re-entry: full GPU parity, smoke, bench (C3), launch list of the bench
O=gpurun_out/r02f; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rA > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err; echo "exit=$?" >> $O/bench_ref.err
