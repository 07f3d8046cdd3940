#!/bin/bash
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batched.py -q -x --timeout 800 > gpurun_out/pytest_batched_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_batched_$TAG.log
tail -30 gpurun_out/pytest_batched_$TAG.log
python scripts/batched_time.py > gpurun_out/batched_time_$TAG.json 2>&1; cat gpurun_out/batched_time_$TAG.json
