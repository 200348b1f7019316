#!/bin/bash
# CPQR v3 check: C3 timing (v1 vs v3), parity suite, then the clock64 trace build
O=gpurun_out/${1:-r02h}; mkdir -p $O
SPQ_CPQR_V1=1 timeout 300 python tools/run_config.py C3 - 6 > $O/c3_v1.log 2>&1
timeout 300 python tools/run_config.py C3 - 6 > $O/c3_v3.log 2>&1
SPQ_CPQR_NTMIN=256 timeout 300 python tools/run_config.py C3 - 6 > $O/c3_v3_nt256.log 2>&1
SPQ_CPQR_NTMIN=512 timeout 300 python tools/run_config.py C3 - 6 > $O/c3_v3_nt512.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
SPQ_TRACE=1 python -m paper_2010_06807_b200.build --force > $O/build.log 2>&1
timeout 300 python tools/cpqr_trace.py > $O/cpqr_trace.txt 2> $O/cpqr_trace.err; echo "exit=$?" >> $O/cpqr_trace.txt
