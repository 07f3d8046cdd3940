"""Solver callers on the device: ACG on the 27-point
stencil and APM on an Erdos-Renyi Laplacian; wall time per iteration (each
iteration = SpMV + 2 qdot + vector updates, one host sync per qdot)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2105_00115_b200 import apps

out = []
for nx in (32, 64, 128):
    a, b = apps.gen_stencil(nx, nx, nx)
    apps.acg(a, b, tau=1e-8, epsilon=1e-8, max_iters=3)          # warm (graphs, device copy)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = apps.acg(a, b, tau=1e-8, epsilon=1e-8)
    dt = time.perf_counter() - t0
    out.append({"solver": "acg", "problem": f"stencil {nx}^3", "n": a.n, "nnz": int(a.csr().nnz),
                "iterations": res.iterations, "s": dt, "us_per_iter": dt / max(res.iterations, 1) * 1e6,
                "converged": res.converged})
    print(json.dumps(out[-1]), flush=True)
for n, p in ((2000, 0.01), (20000, 0.0005)):
    lap = apps.gen_graph_laplacian(n, p, seed=3)
    x0 = np.random.default_rng(4).standard_normal(n)
    apps.apm(lap, x0, tau=1e-6, epsilon=1e-7, max_iters=3)
    t0 = time.perf_counter()
    res = apps.apm(lap, x0, tau=1e-6, epsilon=1e-7, max_iters=300)
    dt = time.perf_counter() - t0
    out.append({"solver": "apm", "problem": f"laplacian n={n} p={p}", "n": n, "nnz": int(lap.csr().nnz),
                "iterations": res.iterations, "s": dt, "us_per_iter": dt / max(res.iterations, 1) * 1e6,
                "converged": res.converged})
    print(json.dumps(out[-1]), flush=True)
