#!/bin/bash
# build the library sources with -DQDOT_SCORE_PROFILE into a standalone binary
# and print the phase clocks of the score CTA
set -e
cd "$(dirname "$0")/.."
C=paper_2105_00115_b200/csrc
mkdir -p /tmp/score_prof
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -DQDOT_SCORE_PROFILE -Iinclude \
  $C/qdot_kernels.cu $C/qdot_capi.cu $C/qdot_apps.cu $C/qdot_exact.cu $C/qdot_host.cu $C/qdot_order.cu $C/qdot_gen.cu \
  scripts/score_prof.cu -o /tmp/score_prof/score_prof
for a in "$@"; do /tmp/score_prof/score_prof $a; done
