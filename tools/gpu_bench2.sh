mkdir -p gpurun_out/b2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b2/bench.json 2> gpurun_out/b2/bench.err; echo "exit=$?" >> gpurun_out/b2/bench.err
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 1500 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x --clock-control none -c 4500 --csv --log-file gpurun_out/b2/launches.csv $CMD > gpurun_out/b2/ncu.log 2>&1
echo "exit=$?" >> gpurun_out/b2/ncu.log
