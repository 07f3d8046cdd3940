#!/bin/bash
# Session check: smoke, GPU tests (not slow), short bench, batched timing + ncu of k_batched.
TAG=${1:-s}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x --timeout 600 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 100 --warmup 5 --e2e-steps 1 --cpu-sample 4194304 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python scripts/batched_time.py > gpurun_out/batched_time_$TAG.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batched -s 3 -c 1 \
   -o gpurun_out/batched_$TAG python scripts/batched_time.py > gpurun_out/ncu_batched_$TAG.log 2>&1
tail -3 gpurun_out/pytest_$TAG.log; cat gpurun_out/bench_$TAG.json gpurun_out/batched_time_$TAG.json
echo done
