#!/bin/bash
# Batched qdot: GPU parity tests, C4 timing, optional ncu capture (NCU=1).
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batched.py -q -x --timeout 800 > gpurun_out/pytest_batched_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_batched_$TAG.log
tail -5 gpurun_out/pytest_batched_$TAG.log
timeout 300 python scripts/batched_time.py > gpurun_out/batched_time_$TAG.json 2>&1; cat gpurun_out/batched_time_$TAG.json
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batched -s 3 -c 1 \
   -o gpurun_out/batched_$TAG python scripts/batched_time.py > gpurun_out/ncu_batched_$TAG.log 2>&1
fi
echo done
