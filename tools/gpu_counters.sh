# per-launch ncu counters of one bench step (cold-cache, serialised):
# duration, DRAM bytes, DMMA / FP64 pipe activity -> profiles/ tables
mkdir -p gpurun_out/ct
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/ct/plain.json 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg,launch__grid_size --clock-control none -c 4500 --csv --log-file gpurun_out/ct/counters.csv $CMD > gpurun_out/ct/ncu.log 2>&1
echo "exit=$?" >> gpurun_out/ct/ncu.log
