"""Where the host time of a small qdot() call goes (cProfile over 2000 calls)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_00115_b200 as Q
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
x = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.randn(n, dtype=torch.float64, device="cuda")
cfg = Q.ToleranceConfig(1e-8)
for _ in range(50):
    Q.qdot(x, y, cfg)
pr = cProfile.Profile()
pr.enable()
for _ in range(2000):
    r = Q.qdot(x, y, cfg)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
