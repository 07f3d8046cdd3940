import time, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2105_00115_b200 import apps
for rep in range(3):
    for nx in (32, 64):
        a, b = apps.gen_stencil(nx, nx, nx)
        orig = apps._IterGraph.capture
        tc = [0.0]
        def cap(self, body, orig=orig):
            t0 = time.perf_counter(); g = orig(self, body); tc[0] += time.perf_counter() - t0; return g
        apps._IterGraph.capture = cap
        torch.cuda.synchronize(); t0 = time.perf_counter()
        res = apps.acg(a, b, tau=1e-8, epsilon=1e-8)
        dt = time.perf_counter() - t0
        apps._IterGraph.capture = orig
        print(rep, nx, res.iterations, f"total {dt*1e3:.1f} ms capture {tc[0]*1e3:.1f} ms per-iter {(dt-tc[0])/res.iterations*1e6:.0f} us", flush=True)
