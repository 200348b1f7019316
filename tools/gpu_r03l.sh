#!/bin/bash
# reflector scalars with fewer fp64 instructions: same-box A/B (two builds), then parity on the default build
O=gpurun_out/${1:-r03l}; mkdir -p $O
for rep in 1 2; do
  SPQ_PLAIN_SCALARS=1 python -m paper_2010_06807_b200.build --force > $O/build_plain.log 2>&1
  python tools/stall_probe.py > $O/calls_plain_$rep.txt 2>&1
  python -m paper_2010_06807_b200.build --force > $O/build_fast.log 2>&1
  python tools/stall_probe.py > $O/calls_fast_$rep.txt 2>&1
done
for f in $O/calls_*.txt; do echo "$(basename $f) $(head -1 $f | cut -c1-28) $(tail -1 $f)"; done > $O/summary.txt
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
