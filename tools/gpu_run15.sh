mkdir -p gpurun_out
for n in 40 44 48; do timeout 900 python tools/diag_levels.py C5 $n > gpurun_out/lev$n.log 2>&1; done
