#!/bin/bash
# C3 / C4 solve timing repeats (noise check) + forced-split parity
O=gpurun_out/${1:-split2}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "split or chain or gmres or unscaled" > $O/pytest_split.log 2>&1; echo "pytest exit=$?" >> $O/pytest_split.log
tail -3 $O/pytest_split.log
for i in 1 2 3; do python tools/solve_timing.py C3 > $O/solve_timing_C3_$i.json 2>/dev/null; done
python tools/solve_timing.py C4 > $O/solve_timing_C4.json 2>/dev/null
python - <<PY
import json
for f in ("C3_1", "C3_2", "C3_3", "C4"):
    d = json.load(open("$O/solve_timing_%s.json" % f))
    print(f, d["solve_w_program"]["waves"], {k: round(v, 3) for k, v in d.items() if k.endswith("device_ms") or k in ("gmres_s",)}, d["gmres_its"], "%.1e" % d["final_res"])
PY
