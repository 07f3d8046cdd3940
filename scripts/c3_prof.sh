#!/bin/bash
# C3 (ill-conditioned, eps 1e-12): pass-1 timing + one ncu --set full capture of k_pass1 (NCU=1).
TAG=${1:-x}
mkdir -p gpurun_out
timeout 300 python scripts/p1_time.py --data illcond --eps 1e-12 > gpurun_out/c3_time_$TAG.json 2>&1; cat gpurun_out/c3_time_$TAG.json
timeout 300 python scripts/p1_time.py --data normal --eps 1e-8 > gpurun_out/c2_time_$TAG.json 2>&1; cat gpurun_out/c2_time_$TAG.json
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 3 -c 1 \
   -o gpurun_out/c3pass1_$TAG python scripts/p1_time.py --data illcond --eps 1e-12 --reps 2 > gpurun_out/ncu_c3_$TAG.log 2>&1
fi
echo done
