"""Small-n latency breakdown: host enqueue cost of the 5 C-ABI calls, GPU drain
rate when enqueue runs ahead, and the fetch (D2H + sync)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_00115_b200 as Q
from paper_2105_00115_b200 import _lib
from paper_2105_00115_b200.device import config_struct, thread_state
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
dev = torch.device("cuda", 0)
x = torch.randn(n, dtype=torch.float64, device=dev)
y = torch.randn(n, dtype=torch.float64, device=dev)
lib = _lib.load()
st = thread_state(dev)
c = config_struct(Q.ToleranceConfig(1e-8), Q.ExactBinning())
s = torch.cuda.current_stream().cuda_stream
ws = st.ws_ptr
cr = ctypes.byref(c)


def enq():
    lib.qdot_b200_begin(ws, s)
    lib.qdot_b200_pass1(x.data_ptr(), y.data_ptr(), n, 0, cr, n, ws, s)
    lib.qdot_b200_score_finalize(ws, n, cr, s)
    lib.qdot_b200_pass2(x.data_ptr(), y.data_ptr(), n, 0, ws, s)
    lib.qdot_b200_finalize(ws, s)


for _ in range(50):
    enq()
torch.cuda.synchronize()
R = 500
t0 = time.perf_counter()
for _ in range(R):
    enq()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"n={n} enqueue-only {(t1 - t0) / R * 1e6:.1f} us/call; pipelined (GPU-bound) {(t2 - t0) / R * 1e6:.1f} us/call")
t0 = time.perf_counter()
for _ in range(R):
    lib.qdot_b200_fetch(ws, ctypes.byref(st.result), st.bins, 4196, s)
print(f"fetch alone {(time.perf_counter() - t0) / R * 1e6:.1f} us")
t0 = time.perf_counter()
for _ in range(R):
    enq()
    lib.qdot_b200_fetch(ws, ctypes.byref(st.result), st.bins, 4196, s)
print(f"enqueue + fetch (synchronous call) {(time.perf_counter() - t0) / R * 1e6:.1f} us")
t0 = time.perf_counter()
for _ in range(R):
    lib.qdot_b200_dot(x.data_ptr(), y.data_ptr(), n, 0, cr, ws, ctypes.byref(st.result), st.bins, 4196, s)
print(f"qdot_b200_dot one call {(time.perf_counter() - t0) / R * 1e6:.1f} us")
