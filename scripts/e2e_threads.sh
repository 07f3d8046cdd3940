#!/bin/bash
# e2e through qdot() from numpy (pageable) inputs vs the staging copy-pool size
for t in 2 4 8 12 16; do
  QDOT_B200_COPY_THREADS=$t python - <<'PY'
import os, sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2105_00115_b200 as Q
n = 1 << 28
rng = np.random.default_rng(0)
x = rng.standard_normal(n); y = rng.standard_normal(n)
cfg = Q.ToleranceConfig(1e-8)
Q.qdot(x, y, cfg); Q.qdot(x, y, cfg)
ts = []
for _ in range(4):
    t0 = time.perf_counter(); Q.qdot(x, y, cfg); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print(os.environ["QDOT_B200_COPY_THREADS"], "threads: best %.1f ms median %.1f ms" % (min(ts) * 1e3, sorted(ts)[2] * 1e3), flush=True)
PY
done
