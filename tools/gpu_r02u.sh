#!/bin/bash
# CPQR v3 A/B: elements per thread (variants 3 = (16,1), 4 = (8,2)) and CTA size; small-interface step trace
O=gpurun_out/${1:-r02u}; mkdir -p $O
run() { tag=$1; shift; env "$@" timeout 300 python tools/run_config.py C3 - 4 > $O/c3_$tag.log 2>&1; }
run default SPQ_X=1
for v in 3 4; do for nt in 128 256 512; do run var${v}_nt${nt} SPQ_CPQR_NVAR=5 SPQ_CPQR_VAR=$v SPQ_CPQR_NTMIN=$nt; done; done
run var0_nt64 SPQ_CPQR_VAR=0 SPQ_CPQR_NTMIN=64
run var0_cl8 SPQ_CPQR_VAR=0 SPQ_CPQR_CLMAX=8
for f in $O/c3_*.log; do echo "$(basename $f) $(grep -E 'level (7|6|5|4|3|2):' $f | grep -oE 'cpqr=[0-9.]+' | tr '\n' ' ') $(grep -E '^factor' $f | tail -2 | tr '\n' ' ')"; done > $O/summary.txt
SPQ_TRACE=1 SPQ_TRACE_MMAX=64 python -m paper_2010_06807_b200.build --force > $O/build.log 2>&1
timeout 300 python tools/cpqr_trace.py > $O/cpqr_trace_small.txt 2> $O/cpqr_trace.err; echo "exit=$?" >> $O/cpqr_trace_small.txt
