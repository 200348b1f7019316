#!/bin/bash
# chunk-size sweep of the solve chains at C4 (larger k: the single-CTA partial reduction grows with the chunk count)
O=gpurun_out/${1:-chainmc4}; mkdir -p $O
for mc in 32 64 128 256; do
  SPQ_CHAIN_MINCHUNK=$mc python tools/solve_timing.py C4 > $O/solve_timing_C4_mc$mc.json 2>/dev/null
done
python - <<PY
import json
for mc in (32, 64, 128, 256):
    d = json.load(open("$O/solve_timing_C4_mc%d.json" % mc))
    print(mc, {k: round(v, 3) for k, v in d.items() if k.endswith("device_ms") or k == "gmres_s"})
PY
