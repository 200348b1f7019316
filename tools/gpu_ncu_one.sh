# full ncu capture of one launch of a kernel (regex $1, skip $2) in one bench step
mkdir -p gpurun_out/nc
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
$CMD > gpurun_out/nc/plain.json 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/nc/$3 $CMD > gpurun_out/nc/$3.log 2>&1
echo "exit=$?" >> gpurun_out/nc/$3.log
