#!/bin/bash
# one compute-sanitizer tool per call: bash tools/gpu_sanitize.sh memcheck|racecheck|synccheck [extra env]
T=${1:-memcheck}; O=gpurun_out/sanitize; mkdir -p $O
timeout 300 python tools/sanitize_cases.py > $O/plain_$T.log 2>&1; echo "plain exit=$?" >> $O/plain_$T.log
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $T --print-limit 50 --error-exitcode 9 \
  python tools/sanitize_cases.py ${2:-} > $O/$T.log 2>&1; echo "sanitizer exit=$?" >> $O/$T.log
tail -5 $O/$T.log
