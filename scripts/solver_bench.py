"""Solver callers on the device: ACG on the 27-point
stencil and APM on an Erdos-Renyi Laplacian; wall time per iteration (each
iteration = SpMV + 2 qdot + vector updates, one host sync per qdot).  Each
solve is repeated REPS times (host jitter dominates single 5-10 ms solves):
median and min per iteration."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2105_00115_b200 import apps

out = []
REPS = int(os.environ.get("REPS", "5"))


def timed(fn):
    ts, res = [], None
    for _ in range(REPS):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = fn()
        ts.append(time.perf_counter() - t0)
    return res, statistics.median(ts), min(ts)
for nx in (32, 64, 128):
    a, b = apps.gen_stencil(nx, nx, nx)
    apps.acg(a, b, tau=1e-8, epsilon=1e-8, max_iters=3)          # warm (graphs, device copy)
    res, dt, dmin = timed(lambda: apps.acg(a, b, tau=1e-8, epsilon=1e-8))
    it = max(res.iterations, 1)
    out.append({"solver": "acg", "problem": f"stencil {nx}^3", "n": a.n, "nnz": int(a.csr().nnz),
                "iterations": res.iterations, "s": dt, "us_per_iter": dt / it * 1e6, "us_per_iter_min": dmin / it * 1e6,
                "reps": REPS, "converged": res.converged})
    print(json.dumps(out[-1]), flush=True)
for n, p in ((2000, 0.01), (20000, 0.0005)):
    lap = apps.gen_graph_laplacian(n, p, seed=3)
    x0 = np.random.default_rng(4).standard_normal(n)
    apps.apm(lap, x0, tau=1e-6, epsilon=1e-7, max_iters=3)
    res, dt, dmin = timed(lambda: apps.apm(lap, x0, tau=1e-6, epsilon=1e-7, max_iters=300))
    it = max(res.iterations, 1)
    out.append({"solver": "apm", "problem": f"laplacian n={n} p={p}", "n": n, "nnz": int(lap.csr().nnz),
                "iterations": res.iterations, "s": dt, "us_per_iter": dt / it * 1e6, "us_per_iter_min": dmin / it * 1e6,
                "reps": REPS, "converged": res.converged})
    print(json.dumps(out[-1]), flush=True)
