#!/bin/bash
# A/B pass-1 timings of library variants (variants/*.so copied over the product lib in turn)
TAG=${1:-ab}; shift
mkdir -p gpurun_out
LIB=paper_2105_00115_b200/lib/libqdot_b200.so
cp $LIB /tmp/prod.so
for v in "$@"; do
  cp variants/$v.so $LIB
  for a in "--norm" "" "--data illcond --eps 1e-12"; do echo "{\"lib\": \"$v\", \"args\": \"$a\"}"; python scripts/p1_time.py $a; done
done > gpurun_out/ab_$TAG.jsonl 2>&1
cp /tmp/prod.so $LIB
cat gpurun_out/ab_$TAG.jsonl
