#!/bin/bash
TAG=${1:-x}
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bw_probe tools/bw_probe.cu && /tmp/bw_probe > gpurun_out/bw_probe_$TAG.jsonl 2>&1
cat gpurun_out/bw_probe_$TAG.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 2 -c 1 \
   -o gpurun_out/pass1_$TAG python scripts/p1_time.py --mode 0 --reps 3 > gpurun_out/ncu_pass1_$TAG.log 2>&1
python scripts/p1_time.py --mode 0
