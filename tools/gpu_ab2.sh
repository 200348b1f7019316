#!/bin/bash
# same-box A/B: interleaved runs of a baseline and a variant (env), C3 timings x2 each + fast tests
O=gpurun_out/${1:-ab}; mkdir -p $O
for rep in 1 2; do
  SPQ_TIMINGS=1 timeout 300 python tools/run_config.py C3 - 3 > $O/c3_a$rep.log 2>&1
  env $2 SPQ_TIMINGS=1 timeout 300 python tools/run_config.py C3 - 3 > $O/c3_b$rep.log 2>&1
done
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > $O/pytest.log 2>&1; echo "exit=$?" >> $O/pytest.log
