#!/bin/bash
LIB=paper_2105_00115_b200/lib/libqdot_b200.so
cp $LIB /tmp/prod.so
cp variants/P_probe_stat.so $LIB
for a in "--norm" ""; do echo "{\"lib\": \"probe\", \"args\": \"$a\"}"; python scripts/p1_time.py $a; done > gpurun_out/probe.jsonl 2>&1
cp variants/P_probe_stat_tune.so $LIB
for v in 1 3 5 6 12 13; do for a in "--norm" ""; do echo "{\"lib\": \"probe_tune\", \"v\": $v, \"args\": \"$a\"}"; QDOT_B200_P1_VARIANT=$v python scripts/p1_time.py $a; done; done >> gpurun_out/probe.jsonl 2>&1
cp /tmp/prod.so $LIB
