mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3200 --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list exit=$?" >> gpurun_out/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cpqr_kernel -s 20 -c 1 -o gpurun_out/prof_cpqr $CMD > gpurun_out/ncu_cpqr.log 2>&1
echo "cpqr exit=$?" >> gpurun_out/ncu_cpqr.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_qr_kernel -s 30 -c 1 -o gpurun_out/prof_panel $CMD > gpurun_out/ncu_panel.log 2>&1
echo "panel exit=$?" >> gpurun_out/ncu_panel.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma2 -s 400 -c 2 -o gpurun_out/prof_gemm $CMD > gpurun_out/ncu_gemm.log 2>&1
echo "gemm exit=$?" >> gpurun_out/ncu_gemm.log
