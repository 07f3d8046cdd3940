#!/bin/bash
# pass-1 variant sweep: gpu_tune.sh TAG LIBVARIANT "variants" "args"
TAG=$1; LV=$2; VS=$3; ARGS=$4
LIB=paper_2105_00115_b200/lib/libqdot_b200.so
cp $LIB /tmp/prod.so; cp variants/$LV.so $LIB
for v in $VS; do echo "{\"lib\": \"$LV\", \"v\": $v, \"args\": \"$ARGS\"}"; QDOT_B200_P1_VARIANT=$v timeout 120 python scripts/p1_time.py $ARGS; done >> gpurun_out/tune_$TAG.jsonl 2>&1
cp /tmp/prod.so $LIB
