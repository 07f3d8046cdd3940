"""ACG / APM cost split: fixed per-solve cost (setup, first r.r, result copy)
versus the marginal cost of one iteration, from solves capped at different
max_iters on the same matrix (graphs already captured)."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2105_00115_b200 import apps


def t_solve(fn, reps=7):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


for nx in (32, 64):
    a, b = apps.gen_stencil(nx, nx, nx)
    apps.acg(a, b, tau=1e-8, epsilon=1e-8, max_iters=3)
    apps.acg(a, b, tau=1e-8, epsilon=1e-8, max_iters=3)
    t1 = t_solve(lambda: apps.acg(a, b, tau=1e-8, epsilon=1e-8, max_iters=1))
    tn = t_solve(lambda: apps.acg(a, b, tau=1e-8, epsilon=1e-8, max_iters=40))
    print(json.dumps({"solver": "acg", "n": a.n, "t_1iter_us": t1 * 1e6, "t_40iter_us": tn * 1e6,
                      "marginal_us_per_iter": (tn - t1) / 39 * 1e6, "fixed_us": (t1 - (tn - t1) / 39) * 1e6}), flush=True)
for n, p in ((2000, 0.01),):
    lap = apps.gen_graph_laplacian(n, p, seed=3)
    x0 = np.random.default_rng(4).standard_normal(n)
    apps.apm(lap, x0, tau=0.0, epsilon=1e-7, max_iters=3)
    apps.apm(lap, x0, tau=0.0, epsilon=1e-7, max_iters=3)
    t1 = t_solve(lambda: apps.apm(lap, x0, tau=0.0, epsilon=1e-7, max_iters=2))
    tn = t_solve(lambda: apps.apm(lap, x0, tau=0.0, epsilon=1e-7, max_iters=41))
    print(json.dumps({"solver": "apm", "n": n, "marginal_us_per_iter": (tn - t1) / 39 * 1e6,
                      "fixed_us": (t1 - 2 * (tn - t1) / 39) * 1e6}), flush=True)
