#!/bin/bash
# host sampling profile of C3 factorizations (library rebuilt with tools/hostprof.cu linked in)
O=gpurun_out/${1:-hp}; mkdir -p $O
SPQ_BUILD_HOSTPROF=1 python -m paper_2010_06807_b200.build --force > $O/build.log 2>&1
SPQ_HOST_PROFILE=$O/hp.txt timeout 300 python tools/run_config.py C3 - 8 > $O/c3.log 2>&1; echo "exit=$?" >> $O/c3.log
python tools/hostprof.py $O/hp.txt 45 > $O/hp_summary.txt 2>&1
python tools/hostprof_lines.py $O/hp.txt > $O/hp_lines.txt 2>&1
