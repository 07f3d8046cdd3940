#!/bin/bash
# full round-end check: smoke, all GPU tests incl. slow, bench (b200 + reference arm)
TAG=${1:-r2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
( time timeout 3000 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 2800 ) > gpurun_out/pytest_full_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
tail -4 gpurun_out/smoke_$TAG.log; tail -6 gpurun_out/pytest_full_$TAG.log; cat gpurun_out/bench_$TAG.json gpurun_out/bench_ref_$TAG.json
