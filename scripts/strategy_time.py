"""Whole qdot step at 2^28 (device inputs) for each binning strategy / tolerance:
shows when pass 2 runs and what it costs."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_00115_b200 as Q
from paper_2105_00115_b200.kernel import run_device
dev = torch.device("cuda", 0)
n = 1 << 28
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
y = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
for strat in ("exact", "ranged:2", "ranged:8", "split:3", "split:6"):
    for eps in (1e-8, 1e-4):
        cfg = Q.ToleranceConfig(eps)
        s = Q.parse_strategy(strat)
        for _ in range(2):
            res, _, _ = run_device(x, y, n, False, cfg, s, timing=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            res, _, _ = run_device(x, y, n, False, cfg, s, timing=False)
        e1.record(); torch.cuda.synchronize()
        print(json.dumps({"strategy": strat, "eps": eps, "ms": e0.elapsed_time(e1) / 5, "pass2_mode": int(res.pass2_needed),
                          "counts": list(res.counts), "n_bins": res.n_bins}), flush=True)
