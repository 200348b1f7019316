# full round-end check: gpu tests (as the driver runs them), smoke, bench
mkdir -p gpurun_out/chk
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/chk/smi.txt 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/chk/tests.log 2>&1; echo "exit=$?" >> gpurun_out/chk/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk/smoke.log 2>&1; echo "exit=$?" >> gpurun_out/chk/smoke.log
timeout 900 python bench.py > gpurun_out/chk/bench.json 2> gpurun_out/chk/bench.err; echo "exit=$?" >> gpurun_out/chk/bench.err
