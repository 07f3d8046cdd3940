#!/bin/bash
# pass-1 iteration: parity tests of the single-vector path + pass-1 timings (dot, norm, C3)
TAG=${1:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_order.py -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
for a in "--norm" "" "--data illcond --eps 1e-12"; do python scripts/p1_time.py $a; done > gpurun_out/p1_$TAG.jsonl 2>&1
tail -3 gpurun_out/pytest_$TAG.log; cat gpurun_out/p1_$TAG.jsonl
