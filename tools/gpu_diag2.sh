#!/bin/bash
# configs sweep + host profile of C3 + ncu --set full of the latency-bound kernels
O=gpurun_out/${1:-d2}; mkdir -p $O
bash tools/gpu_ncu_k.sh ${1:-d2}/nk
bash tools/gpu_hostprof.sh ${1:-d2}/hp
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
bash tools/gpu_configs.sh ${1:-d2}/cfg
