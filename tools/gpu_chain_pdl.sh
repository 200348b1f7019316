#!/bin/bash
# programmatic dependent launch A/B on the solve chains + parity of the solve paths
O=gpurun_out/${1:-chainpdl}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "chain or gmres or solve or golden or variant or unscaled or records" > $O/pytest_chain.log 2>&1; echo "pytest exit=$?" >> $O/pytest_chain.log
tail -3 $O/pytest_chain.log
python tools/solve_timing.py C3 > $O/solve_timing_pdl.json 2>$O/err_pdl.txt
SPQ_CHAIN_NO_DINV=1 python tools/solve_timing.py C3 > $O/solve_timing_nodinv.json 2>/dev/null
SPQ_CHAIN_NO_PDL=1 python tools/solve_timing.py C3 > $O/solve_timing_nopdl.json 2>/dev/null
python tools/solve_timing.py C3 > $O/solve_timing_pdl2.json 2>/dev/null
python - <<PY
import json
for f in ("pdl", "nodinv", "nopdl", "pdl2"):
    d = json.load(open("$O/solve_timing_%s.json" % f))
    print(f, {k: round(v, 3) for k, v in d.items() if k.endswith("device_ms") or k in ("gmres_s", "final_res")})
PY
