import ctypes, json, os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2105_00115_b200 as Q
from paper_2105_00115_b200 import _lib, exact
from paper_2105_00115_b200.device import stream_handle, config_struct, thread_state
dev = torch.device("cuda", 0)
n = 1 << 28
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
y = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
lib = _lib.load(); s = stream_handle(dev); ws = exact._ExactWs(dev)
st = thread_state(dev); c = config_struct(Q.ToleranceConfig(1e-8), Q.ExactBinning())
def ex():
    lib.qdot_b200_exact_accumulate(x.data_ptr(), y.data_ptr(), n, 0, ws.ptr, s)
def p1():
    lib.qdot_b200_pass1(x.data_ptr(), y.data_ptr(), n, 0, ctypes.byref(c), n, st.ws_ptr, s)
def probe():
    lib.qdot_b200_read_probe(x.data_ptr(), n, ws.ptr, s); lib.qdot_b200_read_probe(y.data_ptr(), n, ws.ptr, s)
for name, f in (("exact", ex), ("pass1", p1), ("probe", probe), ("exact", ex)):
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    print(name, e0.elapsed_time(e1) / 10)
