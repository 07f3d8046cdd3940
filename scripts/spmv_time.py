"""SpMV time and effective bandwidth on the stencil matrices: the sliced-ELL
kernel (qdot_b200_sell_spmv, default) and the CSR kernel (qdot_b200_csr_spmv)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2105_00115_b200 import apps


def timed(a, x, y):
    for _ in range(3): a.matvec_device(x, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): a.matvec_device(x, out=y)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 20


for nx in (64, 128):
    a, b = apps.gen_stencil(nx, nx, nx)
    x = torch.ones(a.n, dtype=torch.float64, device="cuda")
    y = a.matvec_device(x)
    nnz = int(a.csr().nnz)
    byts = nnz * 12 + a.n * 8 * 3 + (a.n + 1) * 8
    for kernel in ("sell", "csr"):
        if kernel == "csr":
            a._sell = False
        ms = timed(a, x, y)
        print(json.dumps({"kernel": kernel, "n": a.n, "nnz": nnz, "us": ms * 1e3,
                          "GBps_min_traffic": byts / (ms * 1e-3) / 1e9}))
