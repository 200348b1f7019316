#!/bin/bash
# One GPU round: parity tests, smoke, bench (both arms), launch list of one step,
# ncu --set full of the top kernels.
O=gpurun_out/${1:-r}
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "exit=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "exit=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv --log-file $O/launches.csv $CMD > $O/ncu_list.log 2>&1
echo "exit=$?" >> $O/ncu_list.log
CMD1="python tools/run_config.py C3 - 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma2 -s 20 -c 1 -o $O/gemm $CMD1 > $O/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wyf -s 100 -c 1 -o $O/wyf $CMD1 > $O/ncu_wyf.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_tasks -s 200 -c 1 -o $O/copy $CMD1 > $O/ncu_copy.log 2>&1

timeout 900 ncu --set full --clock-control none --import-source on -k regex:cpqr_reg -s 60 -c 1 -o $O/cpqr $CMD1 > $O/ncu_cpqr.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_qr_reg -s 200 -c 1 -o $O/panel $CMD1 > $O/ncu_panel.log 2>&1
SPQ_SCOPE_LOG=$O/c3_scopes.txt timeout 300 python tools/c3_timeline.py C3 > $O/c3tl.log 2>&1
echo done >> $O/ncu_panel.log
