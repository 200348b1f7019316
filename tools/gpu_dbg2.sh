mkdir -p gpurun_out/db2
SPQ_SPEC_DEBUG=1 timeout 600 python tools/run_config.py C4 - 1 > gpurun_out/db2/c4_spec.log 2>&1
SPQ_SPEC_DEBUG=1 timeout 600 python tools/run_config.py C5 48 1 > gpurun_out/db2/c5_48_spec.log 2>&1
timeout 600 python tools/run_config.py C3 - 3 > gpurun_out/db2/c3.log 2>&1
timeout 600 python tools/run_config.py C4 - 2 > gpurun_out/db2/c4.log 2>&1
