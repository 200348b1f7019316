mkdir -p gpurun_out
for sw in SPQ_CPQR_COOP SPQ_CPQR_GMAPS SPQ_RING_SMALL; do
  env $sw=1 SPQ_CPQR_COOP=1 timeout 600 python -m pytest tests/test_gpu_factor.py -q -x --timeout 300 -k "not c4 and not c5" > gpurun_out/t14_$sw.log 2>&1; echo "exit=$?" >> gpurun_out/t14_$sw.log
done
timeout 900 python tools/diag_exact.py C5 48 exact > gpurun_out/diag14.log 2>&1
