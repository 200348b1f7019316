mkdir -p gpurun_out/sp
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_paths.py -x -q -k "not slow and not c5 and not n48_3d" > gpurun_out/sp/tests.log 2>&1; echo "exit=$?" >> gpurun_out/sp/tests.log
timeout 600 python tools/run_config.py C3 - 3 > gpurun_out/sp/c3.log 2>&1
timeout 600 python tools/run_config.py C4 - 2 > gpurun_out/sp/c4.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/sp/bench.json 2> gpurun_out/sp/bench.err
