#!/bin/bash
# CPQR with a scalar warp (v6) vs v3: A/B, parity, bench, step traces
O=gpurun_out/${1:-r02v}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_batched.py -m gpu -q -x > $O/pytest_kernels.log 2>&1; echo "exit=$?" >> $O/pytest_kernels.log
run() { tag=$1; shift; env "$@" timeout 300 python tools/run_config.py C3 - 5 > $O/c3_$tag.log 2>&1; }
run v3 SPQ_CPQR_V3=1
run v6 SPQ_X=1
run v6_nt256 SPQ_CPQR_NTMIN=256
run v3b SPQ_CPQR_V3=1
run v6b SPQ_X=1
for f in $O/c3_*.log; do echo "$(basename $f) $(grep -E 'level (7|6|5|4|3|2):' $f | grep -oE 'cpqr=[0-9.]+' | tr '\n' ' ') $(grep -E '^factor' $f | tail -3 | tr '\n' ' ')"; done > $O/summary.txt
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
SPQ_TRACE=1 python -m paper_2010_06807_b200.build --force > $O/build.log 2>&1
timeout 300 python tools/cpqr_trace.py > $O/cpqr_trace.txt 2> $O/cpqr_trace.err; echo "exit=$?" >> $O/cpqr_trace.txt
