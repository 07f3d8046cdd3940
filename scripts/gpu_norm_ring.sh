#!/bin/bash
TAG=${1:-nr}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "norm" > gpurun_out/pytest_norm_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_norm_$TAG.log
for r in 0 1 0 1; do echo "{\"ring\": $r}"; QDOT_B200_NORM_RING=$r timeout 120 python scripts/p1_time.py --norm; done > gpurun_out/norm_ring_$TAG.jsonl 2>&1
QDOT_B200_NORM_RING=1 timeout 300 python bench.py --norm --steps 20 --warmup 5 --no-cpu-baseline --no-secondary --e2e-steps 0 > gpurun_out/bench_norm_$TAG.json 2>&1
tail -5 gpurun_out/pytest_norm_$TAG.log; paste - - < gpurun_out/norm_ring_$TAG.jsonl; cut -c1-600 gpurun_out/bench_norm_$TAG.json
