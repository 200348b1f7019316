#!/bin/bash
# long-K small-M GEMMs on large tiles + split-K: GEMM table, same-box A/B on C3, parity
O=gpurun_out/${1:-r03k}; mkdir -p $O
python tools/gemm_vs_cublas.py $O/gemm.json > $O/gemm.txt 2>&1
for rep in 1 2; do
  SPQ_GEMM_V1_ALWAYS=1 python tools/stall_probe.py > $O/calls_v1_$rep.txt 2>&1
  python tools/stall_probe.py > $O/calls_new_$rep.txt 2>&1
done
for f in $O/calls_*.txt; do echo "$(basename $f) $(head -1 $f | cut -c1-28) $(tail -1 $f)"; done > $O/summary.txt
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
