#!/bin/bash
# Round-2 baseline: smoke, GPU tests (non-slow), bench (burst + sustained + e2e), norm bench, batched, latency, solver
TAG=${1:-r2a}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x --timeout 800 -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --steps 20 --warmup 5 --norm --no-cpu-baseline --no-secondary > gpurun_out/bench_norm_$TAG.json 2> gpurun_out/bench_norm_$TAG.err
timeout 300 python scripts/batched_time.py > gpurun_out/batched_$TAG.json 2>&1
timeout 300 python scripts/batched_general_time.py > gpurun_out/batched_general_$TAG.json 2>&1
timeout 300 python scripts/latency.py > gpurun_out/latency_$TAG.jsonl 2>&1
timeout 300 python scripts/solver_bench.py > gpurun_out/solver_bench_$TAG.jsonl 2>&1
( for n in 10000 1000000; do timeout 120 python scripts/step_graph_time.py $n; done ) > gpurun_out/step_graph_$TAG.jsonl 2>&1
tail -3 gpurun_out/pytest_$TAG.log; cat gpurun_out/bench_$TAG.json gpurun_out/bench_norm_$TAG.json gpurun_out/batched_$TAG.json gpurun_out/batched_general_$TAG.json gpurun_out/latency_$TAG.jsonl gpurun_out/step_graph_$TAG.jsonl gpurun_out/solver_bench_$TAG.jsonl
echo done
