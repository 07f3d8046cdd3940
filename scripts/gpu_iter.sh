#!/bin/bash
# Iteration: GPU tests (fast subset), bench, pass1 ncu capture.  Outputs in gpurun_out/.
TAG=${1:-it}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x --timeout 600 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 200 --warmup 10 --e2e-steps 2 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 2 -c 1 \
   -o gpurun_out/pass1_$TAG python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_pass1_$TAG.log 2>&1
echo done
