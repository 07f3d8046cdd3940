#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/p1_sweep_${1:-x}.jsonl
: > $OUT
for v in 0 1 2 3; do
  for m in 1 2; do
    QDOT_B200_P1_VARIANT=$v timeout 300 python scripts/p1_time.py --mode $m >> $OUT 2>>gpurun_out/p1_sweep.err
  done
done
QDOT_B200_P1_VARIANT=0 timeout 300 python scripts/p1_time.py --mode 0 --data illcond --eps 1e-12 >> $OUT 2>>gpurun_out/p1_sweep.err
QDOT_B200_P1_VARIANT=2 timeout 300 python scripts/p1_time.py --mode 0 --data illcond --eps 1e-12 >> $OUT 2>>gpurun_out/p1_sweep.err
cat $OUT
