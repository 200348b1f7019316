#!/bin/bash
# precomputed W = V T^T for every WY record (SPQ_CHAIN_W=1) vs the default threshold
O=gpurun_out/${1:-chainw}; mkdir -p $O
python tools/solve_timing.py C3 > $O/solve_timing_base.json 2>/dev/null
SPQ_CHAIN_W=1 python tools/solve_timing.py C3 > $O/solve_timing_w.json 2>$O/err_w.txt
python - <<PY
import json
for f in ("base", "w"):
    d = json.load(open("$O/solve_timing_%s.json" % f))
    print(f, {k: round(v, 3) for k, v in d.items() if k.endswith("device_ms") or k in ("gmres_s", "final_res")})
PY
