"""Where the time of one qdot() call at small n goes (host side)."""
import cProfile, pstats, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_00115_b200 as Q
from paper_2105_00115_b200.kernel import run_device
n = 10000
x = torch.randn(n, dtype=torch.float64, device="cuda"); y = torch.randn(n, dtype=torch.float64, device="cuda")
cfg = Q.ToleranceConfig(1e-8)
for _ in range(50): Q.qdot(x, y, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(500): Q.qdot(x, y, cfg)
print("qdot()", (time.perf_counter() - t0) / 500 * 1e6, "us")
t0 = time.perf_counter()
for _ in range(500): run_device(x, y, n, False, cfg, Q.ExactBinning(), timing=True)
print("run_device(timing=True)", (time.perf_counter() - t0) / 500 * 1e6, "us")
t0 = time.perf_counter()
for _ in range(500): run_device(x, y, n, False, cfg, Q.ExactBinning(), timing=False)
print("run_device(timing=False)", (time.perf_counter() - t0) / 500 * 1e6, "us")
pr = cProfile.Profile(); pr.enable()
for _ in range(300): Q.qdot(x, y, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
