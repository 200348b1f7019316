mkdir -p gpurun_out
SPQ_PANEL_GLOBAL=1 timeout 600 python -m pytest tests/test_gpu_factor.py -q --timeout 300 -k "not c4 and not c5" > gpurun_out/t13_global.log 2>&1; echo "exit=$?" >> gpurun_out/t13_global.log
for n in 32 40 48; do timeout 600 python tools/diag_exact.py C5 $n >> gpurun_out/diag.log 2>&1; done
timeout 600 python tools/diag_exact.py C5 48 exact >> gpurun_out/diag.log 2>&1
SPQ_PANEL_GLOBAL=1 timeout 600 python tools/diag_exact.py C5 32 >> gpurun_out/diag.log 2>&1
