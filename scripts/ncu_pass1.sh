#!/bin/bash
# Full ncu capture of one warm launch of each kernel of the headline step.
mkdir -p gpurun_out
TAG=${1:-r1}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 2 -c 1 \
   -o gpurun_out/pass1_$TAG python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_pass1_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_finalize|k_score" -s 2 -c 2 \
   -o gpurun_out/small_$TAG python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_small_$TAG.log 2>&1
echo done
