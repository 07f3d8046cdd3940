#!/bin/bash
# A/B of k_batched (exact, C4) across library variants
LIB=paper_2105_00115_b200/lib/libqdot_b200.so
cp $LIB /tmp/prod.so
for v in "$@"; do cp variants/$v.so $LIB; echo "{\"lib\": \"$v\"}"; python scripts/batched_strategy_time.py exact 2>&1 | grep kernel_ms; done > gpurun_out/batched_ab.jsonl
cp /tmp/prod.so $LIB
cat gpurun_out/batched_ab.jsonl
