"""Device time of back-to-back qdot steps (begin, pass1, score_finalize,
pass2_finalize) at size n: eager stream launches and a CUDA graph of 20
steps, no events between the kernels.  QDOT_B200_PDL=0 disables programmatic
dependent launch for an A/B."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_00115_b200 as Q
from paper_2105_00115_b200 import _lib
from paper_2105_00115_b200.device import config_struct, thread_state

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
lib = _lib.load()
x = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.randn(n, dtype=torch.float64, device="cuda")
st = thread_state(x.device)
ws = st.ws_ptr
c = config_struct(Q.ToleranceConfig(1e-8), Q.ExactBinning())
cr = ctypes.byref(c)


PIPE = os.environ.get("PIPE", "enqueue")


def step(s):
    if PIPE == "enqueue":        # the product path (one cluster launch at small n)
        lib.qdot_b200_enqueue(x.data_ptr(), y.data_ptr(), n, 0, cr, ws, s)
        return
    lib.qdot_b200_begin(ws, s)
    lib.qdot_b200_pass1(x.data_ptr(), y.data_ptr(), n, 0, cr, n, ws, s)
    lib.qdot_b200_score_finalize(ws, n, cr, s)
    lib.qdot_b200_pass2_finalize(x.data_ptr(), y.data_ptr(), n, 0, ws, s)


cs = torch.cuda.Stream()
sp = cs.cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(cs):
    for _ in range(50):
        step(sp)
    torch.cuda.synchronize()
    R = 200
    e0.record(cs)
    for _ in range(R):
        step(sp)
    e1.record(cs)
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / R * 1e3
    g = torch.cuda.CUDAGraph()
    g.capture_begin()
    for _ in range(20):
        step(sp)
    g.capture_end()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0.record(cs)
    for _ in range(20):
        g.replay()
    e1.record(cs)
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / 400 * 1e3
print(json.dumps({"n": n, "pipe": PIPE, "pdl": os.environ.get("QDOT_B200_PDL", "1"), "eager_us_per_step": eager,
                  "graph_us_per_step": graph}))
