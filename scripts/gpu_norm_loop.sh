#!/bin/bash
# norm-mode exponent-indexed lean loop: A/B timing (mode 0 vs 32), x.y unchanged, parity
TAG=${1:-nl}
mkdir -p gpurun_out
for m in 0 32 0 32; do timeout 120 python scripts/p1_time.py --norm --mode $m; done > gpurun_out/p1_norm_$TAG.jsonl 2>&1
for m in 0; do timeout 120 python scripts/p1_time.py --mode $m; done >> gpurun_out/p1_norm_$TAG.jsonl 2>&1
timeout 120 python scripts/p1_time.py --norm --data illcond --eps 1e-12 >> gpurun_out/p1_norm_$TAG.jsonl 2>&1
timeout 120 python scripts/p1_time.py --norm --data illcond --eps 1e-12 --mode 32 >> gpurun_out/p1_norm_$TAG.jsonl 2>&1
cat gpurun_out/p1_norm_$TAG.jsonl | cut -c1-250
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "norm or golden" 2>&1 | tail -5
