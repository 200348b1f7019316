mkdir -p gpurun_out
run() { echo "== $*" >> gpurun_out/sweep27.log; env "$@" timeout 300 python tools/run_config.py C3 - 2 2>&1 | grep -E "rep 1|device" | tail -2 | cut -c1-260 >> gpurun_out/sweep27.log; }
run X=0
run SPQ_CPQR_CLMAX=0
run SPQ_CPQR_CLMAX=4
run SPQ_CPQR_CLMAX=8
run SPQ_CPQR_CLMAX=0 SPQ_CPQR_GMAX=32
run SPQ_CPQR_CLMAX=0 SPQ_CPQR_GMAX=64
run SPQ_CPQR_CLMAX=0 SPQ_CPQR_COLS_PER_CTA=16
run SPQ_CPQR_CLMAX=0 SPQ_CPQR_COLS_PER_CTA=4
