#!/bin/bash
O=gpurun_out/c5dbg; mkdir -p $O
run() { tag=$1; shift; env "$@" timeout 600 python tools/run_config.py C5 - 1 > $O/$tag.log 2>&1; echo "exit=$?" >> $O/$tag.log; }
run blocking CUDA_LAUNCH_BLOCKING=1
run nows SPQ_CPQR_NOWS=1
run coop SPQ_CPQR_COOP=1
