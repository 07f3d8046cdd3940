#!/bin/bash
# k_batched: timing + ncu --set full with source (summaries written on the box)
TAG=${1:-b}
mkdir -p gpurun_out
python scripts/batched_time.py > gpurun_out/batched_time_$TAG.json 2>&1
R=gpurun_out/batched_$TAG
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batched -s 3 -c 1 -o $R python scripts/batched_time.py > gpurun_out/ncu_batched_$TAG.log 2>&1
python tools/ncu_summary.py $R.ncu-rep $R > /dev/null 2>&1
python tools/sass_hist.py $R.ncu-rep > ${R}_hist.txt 2>&1
ncu -i $R.ncu-rep --page source --csv --print-source sass > ${R}_sass.csv 2>/dev/null; gzip -f ${R}_sass.csv
rm -f $R.ncu-rep
cat gpurun_out/batched_time_$TAG.json
