#!/bin/bash
# Exercise bench.py's multi-rank path on one GPU (gloo, both ranks on cuda:0) and
# compare its value with one device on the concatenated shards.
mkdir -p gpurun_out
N=${N:-16777216}
QDOT_BENCH_TEST_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
   --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --elements $N --steps 5 --warmup 3 --e2e-steps 1 \
   > gpurun_out/multirank.json 2> gpurun_out/multirank.err; echo "torchrun rc=$?"
tail -3 gpurun_out/multirank.err
python - <<PY
import json, numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_2105_00115_b200 as Q
n = $N
parts = [np.random.default_rng(r) for r in range(2)]
xs, ys = [], []
for rng in parts:
    xs.append(rng.standard_normal(n)); ys.append(rng.standard_normal(n))
x = torch.from_numpy(np.concatenate(xs)).cuda(); y = torch.from_numpy(np.concatenate(ys)).cuda()
ref = Q.qdot(x, y, Q.ToleranceConfig(1e-8)).value
d = json.loads(open("gpurun_out/multirank.json").read().strip().splitlines()[-1])
print("multi-rank value_check", d["value_check"], "single-device", ref, "equal", d["value_check"] == ref)
print("n_gpus", d["n_gpus"], "e2e", d["e2e"]["api"], "keys", sorted(d.keys()))
PY
