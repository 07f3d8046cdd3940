"""Per-stage device time of one small qdot (CUDA events between the stages,
pipelined over many calls)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_00115_b200 as Q
from paper_2105_00115_b200 import _lib
from paper_2105_00115_b200.device import config_struct, thread_state
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
dev = torch.device("cuda", 0)
x = torch.randn(n, dtype=torch.float64, device=dev); y = torch.randn(n, dtype=torch.float64, device=dev)
lib = _lib.load(); st = thread_state(dev); c = config_struct(Q.ToleranceConfig(1e-8), Q.ExactBinning())
s = torch.cuda.current_stream(); sp = s.cuda_stream; ws = st.ws_ptr; cr = ctypes.byref(c)
names = ["begin", "pass1", "score+fin", "pass2+fin", "(none)"]
R = 200
evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(R)]
for it in range(R + 20):
    e = evs[it - 20] if it >= 20 else None
    if e: e[0].record(s)
    lib.qdot_b200_begin(ws, sp)
    if e: e[1].record(s)
    lib.qdot_b200_pass1(x.data_ptr(), y.data_ptr(), n, 0, cr, n, ws, sp)
    if e: e[2].record(s)
    lib.qdot_b200_score_finalize(ws, n, cr, sp)
    if e: e[3].record(s)
    lib.qdot_b200_pass2_finalize(x.data_ptr(), y.data_ptr(), n, 0, ws, sp)
    if e: e[4].record(s)
    pass
    if e: e[5].record(s)
torch.cuda.synchronize()
tot = [0.0] * 5
for e in evs:
    for i in range(5):
        tot[i] += e[i].elapsed_time(e[i + 1])
print(f"n={n}", {nm: round(t / R * 1e3, 1) for nm, t in zip(names, tot)}, "us; sum", round(sum(tot) / R * 1e3, 1))
