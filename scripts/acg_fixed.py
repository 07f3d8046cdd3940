"""Host-side cost of one ACG solve's fixed part (prologue and epilogue around
the device loop), step by step with a synchronize after each (stencil 32^3)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2105_00115_b200 import apps

a, b = apps.gen_stencil(32, 32, 32)
for _ in range(3):
    apps.acg(a, b, tau=1e-8, epsilon=1e-8)
n = a.n
dev = torch.device("cuda")
t = {}


def tick(name, fn, reps=20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    t[name] = round((time.perf_counter() - t0) / reps * 1e6, 1)


x = torch.zeros(n, dtype=torch.float64, device=dev)
q = torch.empty_like(x); r = torch.empty_like(x); p = torch.empty_like(x)
dots = apps._Dots(apps.ToleranceConfig(1e-8), apps.ExactBinning())
tick("to_device_b", lambda: apps._to_device(b, n))
bd = apps._to_device(b, n)
tick("matvec", lambda: a.matvec_device(x, out=q))
tick("update", lambda: apps._update(apps._SUB, bd, 1.0, q, r))
tick("copy", lambda: p.copy_(r))
tick("norm_dot", lambda: apps._norm_dot(dots, r))
tick("x_cpu", lambda: x.cpu().numpy())
st = torch.zeros(8, dtype=torch.float64, device=dev)
tick("st_setitem", lambda: st.__setitem__(0, 1.0))
tick("solve_1iter", lambda: apps.acg(a, b, tau=1e-8, epsilon=1e-8, max_iters=1), reps=10)
tick("solve_full", lambda: apps.acg(a, b, tau=1e-8, epsilon=1e-8), reps=10)
print(json.dumps(t))
