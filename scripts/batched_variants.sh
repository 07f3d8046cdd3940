#!/bin/bash
mkdir -p gpurun_out
for v in ${VARIANTS:-0 1 2}; do QDOT_B200_BATCH_VARIANT=$v timeout 300 python scripts/batched_time.py | sed "s/^/var$v /"; done > gpurun_out/batched_var_${1:-x}.txt 2>&1
cat gpurun_out/batched_var_${1:-x}.txt
