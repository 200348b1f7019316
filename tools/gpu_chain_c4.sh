#!/bin/bash
# per-wave chain profile and solve timing at C4 (3D 32^3)
O=gpurun_out/${1:-chainc4}; mkdir -p $O
python tools/chain_profile.py C4 2> $O/chain_waves_C4.txt > /dev/null
python tools/solve_timing.py C4 > $O/solve_timing_C4.json 2> $O/solve_timing_C4.err
tail -1 $O/solve_timing_C4.json
