#!/bin/bash
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x --timeout 600 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
bash scripts/p1_sweep.sh $TAG
