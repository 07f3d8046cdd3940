#!/bin/bash
# norm-mode exponent-indexed lean loop: A/B timing (mode 0 = prefetch 7 tiles, 64 = 3, 128 = 15,
# 192 = 1, 32 = without the loop), x.y unchanged, C3 data, parity; optional ncu of the norm pass 1
TAG=${1:-nl}
mkdir -p gpurun_out
for m in 0 1024 64 1088 192 1216 0 1024; do timeout 120 python scripts/p1_time.py --norm --mode $m; done > gpurun_out/p1_norm_$TAG.jsonl 2>&1
timeout 120 python scripts/p1_time.py >> gpurun_out/p1_norm_$TAG.jsonl 2>&1
timeout 120 python scripts/p1_time.py --norm --data illcond --eps 1e-12 >> gpurun_out/p1_norm_$TAG.jsonl 2>&1
cut -c1-200 gpurun_out/p1_norm_$TAG.jsonl
[ -n "$NCU" ] && bash scripts/gpu_ncu_one.sh pn_$TAG k_pass1 python scripts/p1_time.py --norm --reps 2
[ -n "$TESTS" ] && timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "norm or golden" 2>&1 | tail -2
true
