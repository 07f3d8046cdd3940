#!/bin/bash
# needs a tuning build: NVCC extra flag -DQDOT_B200_P1_TUNING (variants are not in the default library)
mkdir -p gpurun_out
OUT=gpurun_out/p1_sweep_${1:-x}.jsonl
: > $OUT
for v in ${VARIANTS:-0 1 2 3 4 5}; do
  QDOT_B200_P1_VARIANT=$v timeout 300 python scripts/p1_time.py --mode 0 >> $OUT 2>>gpurun_out/p1_sweep.err
done
for v in ${IVARIANTS:-0 3}; do
  QDOT_B200_P1_VARIANT=$v timeout 300 python scripts/p1_time.py --mode 0 --data illcond --eps 1e-12 >> $OUT 2>>gpurun_out/p1_sweep.err
done
cat $OUT
