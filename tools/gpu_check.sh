#!/bin/bash
# Quick check of a host-side change: C3 timings (3 factorizations, twice) with the
# host breakdown, the GPU parity suite, and the default bench line.
O=gpurun_out/${1:-check}; mkdir -p $O
for rep in 1 2; do timeout 300 python tools/c3_timeline.py C3 > $O/c3_$rep.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "exit=$?" >> $O/pytest.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "exit=$?" >> $O/bench.err
timeout 400 python tools/e2e_prof.py > $O/e2e_prof.txt 2>&1
