#!/bin/bash
# bulk-copy candidate exchange for long records: A/B on C3 and C4, parity
O=gpurun_out/${1:-r02x}; mkdir -p $O
run() { cfg=$1; tag=$2; shift 2; env "$@" timeout 600 python tools/run_config.py $cfg - 4 > $O/${cfg}_$tag.log 2>&1; }
run C3 off SPQ_CPQR_BULK_BYTES=100000000
run C3 on SPQ_X=1
run C3 on512 SPQ_CPQR_BULK_BYTES=512
run C4 off SPQ_CPQR_BULK_BYTES=100000000
run C4 on SPQ_X=1
for f in $O/C*.log; do echo "$(basename $f) $(grep -E 'level [0-9]+:' $f | grep -oE 'cpqr=[0-9.]+' | tr '\n' ' ') $(grep -E '^factor' $f | tail -2 | tr '\n' ' ')"; done > $O/summary.txt
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
