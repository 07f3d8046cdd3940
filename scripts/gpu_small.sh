#!/bin/bash
# small-n latency: per-part graph timing, step graph, qdot() latency, solvers
TAG=${1:-sm}
mkdir -p gpurun_out
( for n in 1000 10000 100000; do timeout 120 python scripts/small_parts.py $n; done ) > gpurun_out/small_parts_$TAG.jsonl 2>&1
( for n in 1000 10000 32768 65536 100000 1000000; do timeout 120 python scripts/step_graph_time.py $n; PIPE=four timeout 120 python scripts/step_graph_time.py $n; done ) > gpurun_out/step_graph_$TAG.jsonl 2>&1
timeout 300 python scripts/latency.py > gpurun_out/latency_$TAG.jsonl 2>&1
timeout 300 python scripts/acg_breakdown.py > gpurun_out/acg_breakdown_$TAG.jsonl 2>&1
timeout 300 python scripts/solver_bench.py > gpurun_out/solver_bench_$TAG.jsonl 2>&1
cat gpurun_out/small_parts_$TAG.jsonl gpurun_out/step_graph_$TAG.jsonl gpurun_out/latency_$TAG.jsonl gpurun_out/acg_breakdown_$TAG.jsonl gpurun_out/solver_bench_$TAG.jsonl | cut -c1-300
