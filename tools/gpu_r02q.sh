#!/bin/bash
# copy MLP, flag-check batching, T/W overlap, host micro-opts: A/B + parity + bench + host profile
O=gpurun_out/${1:-r02q}; mkdir -p $O
SPQ_NO_T_OVERLAP=1 timeout 300 python tools/run_config.py C3 - 6 > $O/c3_no_overlap.log 2>&1
timeout 300 python tools/run_config.py C3 - 6 > $O/c3.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
bash tools/gpu_hostprof.sh ${1:-r02q}/hp > /dev/null 2>&1
