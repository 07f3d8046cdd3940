"""Small-n step breakdown: device time per step of CUDA graphs holding subsets
of the qdot pipeline (begin, pass 1, score+finalize, pass 2+finalize) at size
n, 20 steps per graph.  Subsets give wrong results (workspace not reset); only
the timing is used."""
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
parts = {
    "begin": lambda s: lib.qdot_b200_begin(ws, s),
    "pass1": lambda s: lib.qdot_b200_pass1(x.data_ptr(), y.data_ptr(), n, 0, cr, n, ws, s),
    "score": lambda s: lib.qdot_b200_score_finalize(ws, n, cr, s),
    "pass2": lambda s: lib.qdot_b200_pass2_finalize(x.data_ptr(), y.data_ptr(), n, 0, ws, s),
}
combos = [["begin", "pass1", "score", "pass2"], ["pass1", "score", "pass2"], ["begin", "pass1", "score"],
          ["begin"], ["pass1"], ["score"], ["pass2"], ["begin", "pass1"], ["score", "pass2"]]
cs = torch.cuda.Stream()
sp = cs.cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
out = {"n": n}
with torch.cuda.stream(cs):
    for combo in combos:
        for _ in range(5):
            for p in ["begin", "pass1", "score", "pass2"]:
                parts[p](sp)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        g.capture_begin()
        for _ in range(20):
            for p in combo:
                parts[p](sp)
        g.capture_end()
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0.record(cs)
            for _ in range(10):
                g.replay()
            e1.record(cs)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 200 * 1e3)
        out["+".join(combo)] = round(sorted(ts)[2], 2)
print(json.dumps(out))
