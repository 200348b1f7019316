#!/bin/bash
# config-2 and config-5 bench lines (clock-recorded) + the size sweep
O=gpurun_out/r02e; mkdir -p $O
timeout 900 python bench.py --config C2 --steps 5 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err; echo "exit=$?" >> $O/bench_c2.err
timeout 2400 python tools/scaling_sweep.py $O/sweep.json --oracle-budget 60 > $O/sweep.log 2>&1; echo "exit=$?" >> $O/sweep.log
timeout 2400 python bench.py --config C5 --steps 2 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err; echo "exit=$?" >> $O/bench_c5.err
