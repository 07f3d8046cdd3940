#!/bin/bash
# norm-mode pass 1: timing + one ncu --set full capture with source
TAG=${1:-norm}
mkdir -p gpurun_out
python scripts/p1_time.py --norm > gpurun_out/p1_norm_$TAG.json 2>&1
python scripts/p1_time.py > gpurun_out/p1_dot_$TAG.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 3 -c 1 \
   -o gpurun_out/p1norm_$TAG python scripts/p1_time.py --norm --reps 2 > gpurun_out/ncu_p1norm_$TAG.log 2>&1
cat gpurun_out/p1_norm_$TAG.json gpurun_out/p1_dot_$TAG.json; tail -3 gpurun_out/ncu_p1norm_$TAG.log
