mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 280 > gpurun_out/t5.log 2>&1; echo "exit=$?" >> gpurun_out/t5.log
timeout 300 python tools/run_config.py C3 - 3 > gpurun_out/c3_5.log 2>&1; echo "exit=$?" >> gpurun_out/c3_5.log
SPQ_GEMM=1 timeout 300 python tools/fp64_peak.py > gpurun_out/peak_v1.log 2>&1
timeout 300 python tools/fp64_peak.py > gpurun_out/peak_v2.log 2>&1
