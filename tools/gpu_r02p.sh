#!/bin/bash
# round-2 evidence run: size sweep (J3), bench lines of C2 / C1 / C4 / C5 with clocks (J1, J2)
O=gpurun_out/${1:-r02p}; mkdir -p $O
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 > $O/bench_C2.json 2> $O/bench_C2.err; echo "exit=$?" >> $O/bench_C2.err
timeout 600 python bench.py --config C1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C1.json 2> $O/bench_C1.err; echo "exit=$?" >> $O/bench_C1.err
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err; echo "exit=$?" >> $O/bench_C4.err
timeout 1500 python bench.py --config C5 --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err; echo "exit=$?" >> $O/bench_C5.err
(while true; do nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active,power.draw --format=csv,noheader >> $O/sweep_clocks.txt; sleep 5; done) & CL=$!
timeout 2400 python tools/scaling_sweep.py $O/sweep.json --oracle-budget 60 > $O/sweep.log 2>&1; echo "exit=$?" >> $O/sweep.log
kill $CL
