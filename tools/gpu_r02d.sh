#!/bin/bash
O=gpurun_out/r02d; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -rA > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit=$?" >> $O/smoke.log
