#!/bin/bash
# C5 (BASELINE configs[4]): one fixed 2^31-element pair, strong scaling over G
# ranks.  On a one-GPU box the G > 1 runs put every rank on cuda:0 over gloo
# (QDOT_BENCH_TEST_SHARED_GPU=1): the timings of those mean nothing, the
# value_check / bins_hash must be identical for every G.
mkdir -p gpurun_out
N=${N:-2147483648}
for G in 1 2 4 8; do
  if [ "$G" = 1 ]; then
    timeout 900 python bench.py --gpus 1 --n-total $N --steps 5 --warmup 3 --e2e-steps 0 --no-secondary \
      --no-cpu-baseline --sustained-ms 0 > gpurun_out/r2_c5_G$G.json 2> gpurun_out/r2_c5_G$G.err
  else
    QDOT_BENCH_TEST_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
      --master-addr 127.0.0.1 --master-port $((29600 + G)) bench.py --gpus $G --n-total $N --steps 3 --warmup 3 \
      --e2e-steps 0 --no-secondary --no-cpu-baseline --sustained-ms 0 \
      > gpurun_out/r2_c5_G$G.json 2> gpurun_out/r2_c5_G$G.err
  fi
  echo "G=$G rc=$?"
done
python - <<'PY'
import json
rows = []
for g in (1, 2, 4, 8):
    try:
        d = json.loads(open(f"gpurun_out/r2_c5_G{g}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(g, "no output", e); continue
    rows.append((g, d["value_check"], d["bins_hash"], d["n_bins"], d["config"]["n_total"], d["scaling"]))
    print(g, d["value_check"], d["bins_hash"], d["n_bins"], d["config"]["n_per_gpu"], d["ms_per_step"])
print("identical:", len({(r[1], r[2]) for r in rows}) == 1 and len(rows) == 4)
json.dump({"what": "C5 strong scaling, n=2^31 device-generated standard-normal pair, eps 1e-8 exact; "
                   "G>1 emulated on one B200 (gloo, all ranks on cuda:0; timings not meaningful)",
           "rows": [dict(zip(["G", "value_check", "bins_hash", "n_bins", "n_total", "scaling"], r)) for r in rows],
           "identical": len({(r[1], r[2]) for r in rows}) == 1 and len(rows) == 4},
          open("gpurun_out/r2_c5_summary.json", "w"), indent=1)
PY
