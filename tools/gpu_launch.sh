# launch list of one bench step (per-kernel device times), after a plain run
mkdir -p gpurun_out/ll
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/ll/plain.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 5000 --csv --log-file gpurun_out/ll/launches.csv $CMD > gpurun_out/ll/ncu.log 2>&1
echo "exit=$?" >> gpurun_out/ll/ncu.log
