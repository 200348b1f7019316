#!/bin/bash
# chunk-size A/B of the solve chains (SPQ_CHAIN_MINCHUNK)
O=gpurun_out/${1:-chainmc}; mkdir -p $O
for mc in 8 16 24 32; do
  SPQ_CHAIN_MINCHUNK=$mc python tools/solve_timing.py C3 > $O/solve_timing_mc$mc.json 2>/dev/null
done
python - <<PY
import json
for mc in (8, 16, 24, 32):
    d = json.load(open("$O/solve_timing_mc%d.json" % mc))
    print(mc, {k: round(v, 3) for k, v in d.items() if k.endswith("device_ms") or k == "gmres_s"})
PY
