#!/bin/bash
# round-2 A/B: malloc policy, CPQR v1 vs v2, then parity + bench
O=gpurun_out/r02g; mkdir -p $O
SPQ_NO_MALLOPT=1 SPQ_CPQR_V1=1 timeout 300 python tools/run_config.py C3 - 8 > $O/c3_nomallopt_v1.log 2>&1
SPQ_CPQR_V1=1 timeout 300 python tools/run_config.py C3 - 8 > $O/c3_v1.log 2>&1
timeout 300 python tools/run_config.py C3 - 8 > $O/c3_v2.log 2>&1
SPQ_CPQR_LOG=1 timeout 300 python tools/run_config.py C3 - 1 2> $O/cpqr_sizes.txt > /dev/null
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
timeout 300 python tools/solve_timing.py C3 > $O/solve_timing.json 2> $O/solve_timing.err
timeout 300 python tools/chain_profile.py C3 > /dev/null 2> $O/chain_waves.txt
