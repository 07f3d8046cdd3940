"""Time the device exact dot (k_exact) on C2 (2^28 standard normal) and a
C3-like wide-exponent input, CUDA events, plain=False."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_00115_b200 as Q
from paper_2105_00115_b200 import _lib, exact
from paper_2105_00115_b200.device import stream_handle
dev = torch.device("cuda", 0)
n = 1 << 28
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
y = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
lib = _lib.load()
s = stream_handle(dev)
ws = exact._ExactWs(dev)
from oracle.oracle import gen_illcond
xi, yi = gen_illcond(n, seed=0)
cases = {"c2_normal": (x, y), "c3_illcond": (torch.from_numpy(xi).to(dev), torch.from_numpy(yi).to(dev))}
del xi, yi
for name, (a, b) in cases.items():
    def run():
        _lib.check(lib.qdot_b200_exact_begin(ws.ptr, s))
        _lib.check(lib.qdot_b200_exact_accumulate(a.data_ptr(), b.data_ptr(), n, 0, ws.ptr, s))
    for _ in range(3): run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    r = Q.reference_dot(a, b, plain=False)
    print(json.dumps({"kernel": "k_exact", "input": name, "n": n, "ms": ms, "GBps": n * 16 / ms / 1e6, "value": r.value}))
