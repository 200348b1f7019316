#!/bin/bash
# C5 (3D 64^3) on the final code: factorization + device GMRES through the reworked chains
O=gpurun_out/${1:-c5final}; mkdir -p $O
timeout 1700 python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err; echo "exit=$?" >> $O/bench_C5.err
tail -3 $O/bench_C5.err; cut -c1-600 $O/bench_C5.json
