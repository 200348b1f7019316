mkdir -p gpurun_out
for n in 40 48; do
  timeout 600 python tools/run_config.py C5 $n 1 > gpurun_out/c5n$n.log 2>&1; echo "exit=$?" >> gpurun_out/c5n$n.log
done
timeout 1500 python tools/run_config.py C5 - 1 > gpurun_out/c5.log 2>&1; echo "exit=$?" >> gpurun_out/c5.log
