"""Host-side profile of one ACG solve (32^3 stencil) after warm-up."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_00115_b200 import apps
a, b = apps.gen_stencil(32, 32, 32)
apps.acg(a, b, tau=1e-8, epsilon=1e-8, max_iters=3)
apps.acg(a, b, tau=1e-8, epsilon=1e-8)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    apps.acg(a, b, tau=1e-8, epsilon=1e-8)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
