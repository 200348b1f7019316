#!/bin/bash
O=gpurun_out/r02c; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rA -k "not c5 and not n48_3d" > $O/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> $O/pytest_gpu.log
