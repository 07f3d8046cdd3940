import time, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2105_00115_b200 as Q
X = torch.randn(1024, 4096, dtype=torch.float64, device="cuda"); Y = torch.randn(1024, 4096, dtype=torch.float64, device="cuda")
for strat in (Q.ExactBinning(), Q.RangedBinning(3)):
    Q.qdot_batched(X, Y, Q.ToleranceConfig(1e-6), strat)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = Q.qdot_batched(X, Y, Q.ToleranceConfig(1e-6), strat)
    print(type(strat).__name__, (time.perf_counter() - t0) * 1e3, "ms", len(r.general_rows), "general rows")
