#!/bin/bash
# per-kernel device times inside ACG 32^3 iterations (ncu launch list), with the
# cluster qdot path forced on (QDOT_B200_SMALL_AUTO=65536) and off
TAG=${1:-al}
mkdir -p gpurun_out
cat > /tmp/acg_one.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2105_00115_b200 import apps
a, b = apps.gen_stencil(32, 32, 32)
for _ in range(3):
    apps.acg(a, b, tau=1e-8, epsilon=1e-8, max_iters=6)
PY
for mode in small four; do
  if [ $mode = small ]; then export QDOT_B200_SMALL_AUTO=65536; else export QDOT_B200_SMALL_AUTO=1; fi
  timeout 300 ncu --graph-profiling node --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/acg_launch_${mode}_$TAG.csv python /tmp/acg_one.py > /dev/null 2>&1
  python - "$mode" "gpurun_out/acg_launch_${mode}_$TAG.csv" <<'PY'
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[2])))
hdr = None; d = collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        rec = dict(zip(hdr, r))
        if rec.get('Metric Name') == 'gpu__time_duration.sum': d[rec['Kernel Name'][:40]].append(float(rec['Metric Value']))
print(sys.argv[1])
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])): print("  ", len(v), round(sum(v)/len(v)), k)
PY
done
