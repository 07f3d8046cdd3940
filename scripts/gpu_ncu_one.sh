#!/bin/bash
# ncu --set full of one kernel: gpu_ncu_one.sh TAG KERNEL_REGEX CMD...
TAG=$1; K=$2; shift 2
mkdir -p gpurun_out
R=gpurun_out/ncu_$TAG
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $R "$@" > gpurun_out/ncu_${TAG}.log 2>&1
python tools/ncu_summary.py $R.ncu-rep $R > /dev/null 2>&1
python tools/sass_hist.py $R.ncu-rep > ${R}_hist.txt 2>&1
ncu -i $R.ncu-rep --page source --csv --print-source sass > ${R}_sass.csv 2>/dev/null; gzip -f ${R}_sass.csv
[ -n "$KEEP_REP" ] || rm -f $R.ncu-rep
head -30 $R.txt; head -25 ${R}_hist.txt
