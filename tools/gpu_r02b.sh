#!/bin/bash
# parity pass: record-level comparisons against the live reference, unscaled route
O=gpurun_out/r02b; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rA -k "not c5" > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
