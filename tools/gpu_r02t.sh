#!/bin/bash
# blocked larft: A/B on C3, kernel golden tests first, then the full parity suite and a bench
O=gpurun_out/${1:-r02t}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x > $O/pytest_kernels.log 2>&1; echo "exit=$?" >> $O/pytest_kernels.log
SPQ_LARFT_ROWWISE=1 timeout 300 python tools/run_config.py C3 - 6 > $O/c3_rowwise.log 2>&1
timeout 300 python tools/run_config.py C3 - 6 > $O/c3.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench exit=$?" >> $O/bench.err
