#!/bin/bash
TAG=${1:-sm}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python scripts/latency.py > gpurun_out/latency_$TAG.jsonl 2>&1
( for n in 1000 10000 100000 1000000; do timeout 120 python scripts/step_graph_time.py $n; done ) > gpurun_out/step_graph_$TAG.jsonl 2>&1
timeout 300 python scripts/solver_bench.py > gpurun_out/solver_bench_$TAG.jsonl 2>&1
tail -3 gpurun_out/pytest_$TAG.log; cat gpurun_out/latency_$TAG.jsonl gpurun_out/step_graph_$TAG.jsonl gpurun_out/solver_bench_$TAG.jsonl
