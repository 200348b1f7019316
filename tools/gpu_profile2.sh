mkdir -p gpurun_out/p2
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/p2/smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/p2/bench.json 2> gpurun_out/p2/bench.err; echo "exit=$?" >> gpurun_out/p2/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/p2/bench_ref.json 2> gpurun_out/p2/bench_ref.err
timeout 300 python tools/config2.py > gpurun_out/p2/config2.json 2>&1
timeout 600 python tools/run_config.py C4 - 2 > gpurun_out/p2/c4.log 2>&1
timeout 600 python tools/run_config.py C1 - 3 > gpurun_out/p2/c1.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/p2/prof_plain.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv --log-file gpurun_out/p2/launches.csv $CMD > gpurun_out/p2/ncu_list.log 2>&1
echo "list exit=$?" >> gpurun_out/p2/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cpqr_kernel -s 20 -c 1 -o gpurun_out/p2/prof_cpqr $CMD > gpurun_out/p2/ncu_cpqr.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma2_kernel -s 300 -c 2 -o gpurun_out/p2/prof_gemm $CMD > gpurun_out/p2/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_qr -s 40 -c 1 -o gpurun_out/p2/prof_panel $CMD > gpurun_out/p2/ncu_panel.log 2>&1
