#!/bin/bash
# bench step-time outliers: collector pauses? clock sampler?
O=gpurun_out/${1:-r02o}; mkdir -p $O
for tag in plain nogc; do
  if [ $tag = nogc ]; then export SPQ_BENCH_NOGC=1; fi
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$tag.json 2> $O/bench_$tag.err
  python -c "import json;d=json.load(open('$O/bench_$tag.json'));print('$tag',round(d['value'],3),d['step_ms'])" >> $O/summary.txt
done
