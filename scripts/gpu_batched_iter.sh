#!/bin/bash
TAG=${1:-bi}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batched.py -q -x -p no:cacheprovider > gpurun_out/pytest_batched_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_batched_$TAG.log
timeout 300 python scripts/batched_strategy_time.py > gpurun_out/batched_strat_$TAG.jsonl 2>&1
tail -15 gpurun_out/pytest_batched_$TAG.log; cat gpurun_out/batched_strat_$TAG.jsonl
