mkdir -p gpurun_out
timeout 300 python tools/kbench.py > gpurun_out/kbench2.log 2>&1; echo "exit=$?" >> gpurun_out/kbench2.log
for n in 24 32 40 48; do
  timeout 600 python tools/run_config.py C5 $n 1 > gpurun_out/c5n$n.log 2>&1; echo "exit=$?" >> gpurun_out/c5n$n.log
done
