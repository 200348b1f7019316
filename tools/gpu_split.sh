#!/bin/bash
# row-block split of large back substitutions: parity (forced split), C4 solve timing A/B
O=gpurun_out/${1:-split}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "split or chain or gmres or unscaled" > $O/pytest_split.log 2>&1; echo "pytest exit=$?" >> $O/pytest_split.log
tail -15 $O/pytest_split.log
python tools/solve_timing.py C4 > $O/solve_timing_C4_split.json 2> $O/err1.txt
SPQ_CHAIN_NO_SPLIT=1 python tools/solve_timing.py C4 > $O/solve_timing_C4_nosplit.json 2>/dev/null
for s in 128 192 384; do SPQ_CHAIN_SPLIT_K=$s python tools/solve_timing.py C4 > $O/solve_timing_C4_s$s.json 2>/dev/null; done
python tools/solve_timing.py C3 > $O/solve_timing_C3.json 2>/dev/null
python - <<PY
import json
for f in ("C4_split", "C4_nosplit", "C4_s128", "C4_s192", "C4_s384", "C3"):
    try:
        d = json.load(open("$O/solve_timing_%s.json" % f))
        print(f, d["solve_w_program"]["waves"], {k: round(v, 3) for k, v in d.items() if k.endswith("device_ms") or k in ("gmres_s",)}, d["gmres_its"], "%.1e" % d["final_res"])
    except Exception as e:
        print(f, "ERR", e)
PY
