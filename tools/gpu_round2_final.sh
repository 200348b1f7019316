#!/bin/bash
# round-2 closing run: parity, smoke, bench (default arguments and 20 steps, both arms), C2, C3 gaps, launch list
O=gpurun_out/${1:-r02final}; mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench exit=$?" >> $O/bench_default.err
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err; echo "exit=$?" >> $O/bench_ref.err
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 > $O/bench_C2.json 2> $O/bench_C2.err; echo "exit=$?" >> $O/bench_C2.err
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err; echo "exit=$?" >> $O/bench_C4.err
SPQ_SCOPE_LOG=$O/c3_scopes.txt timeout 300 python tools/c3_timeline.py C3 > $O/c3tl.log 2>&1
python tools/timeline_gaps.py $O/c3_scopes.txt 25 > $O/gaps.txt 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "exit=$?" >> $O/ncu_launch.log
