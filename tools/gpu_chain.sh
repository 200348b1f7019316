#!/bin/bash
# chain diagnostics: parity of the solve paths, per-wave times (phase A split), solve timing
O=gpurun_out/${1:-chain}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "chain or gmres or solve or golden or variant or unscaled or records" > $O/pytest_chain.log 2>&1; echo "pytest exit=$?" >> $O/pytest_chain.log
tail -3 $O/pytest_chain.log
python tools/chain_profile.py C3 2> $O/chain_waves.txt > /dev/null
python tools/solve_timing.py C3 > $O/solve_timing.json 2> $O/solve_timing.err
tail -1 $O/solve_timing.json
for mc in 32 128; do
  SPQ_CHAIN_MINCHUNK=$mc python tools/solve_timing.py C3 > $O/solve_timing_mc$mc.json 2>/dev/null
done
python - <<PY
import json
for f in ("solve_timing", "solve_timing_mc32", "solve_timing_mc128"):
    d = json.load(open("$O/%s.json" % f))
    print(f, {k: round(v, 3) for k, v in d.items() if k.endswith("device_ms") or k == "gmres_s"})
PY
