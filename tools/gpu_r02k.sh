#!/bin/bash
# panel QR tail restructure: C3 timing, parity, trace build
O=gpurun_out/${1:-r02k}; mkdir -p $O
timeout 300 python tools/run_config.py C3 - 6 > $O/c3.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
SPQ_TRACE=1 python -m paper_2010_06807_b200.build --force > $O/build.log 2>&1
timeout 300 python tools/panel_trace.py > $O/panel_trace.txt 2>&1; echo "exit=$?" >> $O/panel_trace.txt
timeout 300 python tools/cpqr_trace.py > $O/cpqr_trace.txt 2> $O/cpqr_trace.err; echo "exit=$?" >> $O/cpqr_trace.txt
