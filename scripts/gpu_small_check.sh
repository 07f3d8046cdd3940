#!/bin/bash
# the one-launch cluster path: parity suites that reach it, then small-n timings
TAG=${1:-sc}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_apps.py tests/test_gpu_order.py tests/test_gpu_cli.py -q -x -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_small_$TAG.log
cat gpurun_out/pytest_small_$TAG.log
bash scripts/gpu_small.sh $TAG
