#!/bin/bash
# reserve fix check + C2 line + round evidence: parity, smoke, bench (both arms), ncu launch list, ncu --set full of the top kernels
O=gpurun_out/${1:-r02r}; mkdir -p $O
timeout 300 python tools/run_config.py C3 - 6 > $O/c3.log 2>&1
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 > $O/bench_C2.json 2> $O/bench_C2.err; echo "exit=$?" >> $O/bench_C2.err
timeout 900 python bench.py --steps 20 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err; echo "exit=$?" >> $O/bench_ref.err
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit=$?" >> $O/smoke.log
SPQ_SCOPE_LOG=$O/c3_scopes.txt timeout 300 python tools/c3_timeline.py C3 > $O/c3tl.log 2>&1
python tools/timeline_gaps.py $O/c3_scopes.txt 25 > $O/gaps.txt 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "exit=$?" >> $O/ncu_launch.log
