#!/bin/bash
# clock64 phase breakdown of the latency-bound kernels (diagnostic SPQ_TRACE build on the box only)
O=gpurun_out/${1:-trace}; mkdir -p $O
SPQ_TRACE=1 python -m paper_2010_06807_b200.build --force > $O/build.log 2>&1
timeout 300 python tools/cpqr_trace.py > $O/cpqr_trace.txt 2>&1; echo "exit=$?" >> $O/cpqr_trace.txt
[ -f tools/panel_trace.py ] && { timeout 300 python tools/panel_trace.py > $O/panel_trace.txt 2>&1; echo "exit=$?" >> $O/panel_trace.txt; }
