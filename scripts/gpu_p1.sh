#!/bin/bash
# pass-1 change check: GPU parity (not slow), C2/C3 pass-1 timing, optional ncu of C3 (NCU=1).
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -q -x --timeout 800 > gpurun_out/pytest_p1_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p1_$TAG.log
tail -3 gpurun_out/pytest_p1_$TAG.log
NCU=${NCU:-0} bash scripts/c3_prof.sh $TAG
