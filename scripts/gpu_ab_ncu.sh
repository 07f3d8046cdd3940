#!/bin/bash
# ncu --set full of k_pass1 for library variants: gpu_ab_ncu.sh TAG "ARGS" variant...
TAG=$1; ARGS=$2; shift 2
mkdir -p gpurun_out
LIB=paper_2105_00115_b200/lib/libqdot_b200.so
cp $LIB /tmp/prod.so
for v in "$@"; do
  cp variants/$v.so $LIB
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass1 -s 3 -c 1 \
     -o gpurun_out/p1_${TAG}_$v python scripts/p1_time.py $ARGS --reps 2 > gpurun_out/ncu_p1_${TAG}_$v.log 2>&1
done
cp /tmp/prod.so $LIB
for v in "$@"; do
  R=gpurun_out/p1_${TAG}_$v
  python tools/ncu_summary.py $R.ncu-rep $R > /dev/null 2>&1
  python tools/sass_hist.py $R.ncu-rep > ${R}_hist.txt 2>&1
  ncu -i $R.ncu-rep --page source --csv --print-source sass > ${R}_sass.csv 2>/dev/null
  gzip -f ${R}_sass.csv
  [ -n "$KEEP_REP" ] || rm -f $R.ncu-rep
done
