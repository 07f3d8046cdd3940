"""A few eager qdot steps at small n (for an ncu launch list: per-kernel durations)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_00115_b200 as Q
from paper_2105_00115_b200 import _lib
from paper_2105_00115_b200.device import config_struct, thread_state
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
lib = _lib.load()
x = torch.randn(n, dtype=torch.float64, device="cuda"); y = torch.randn(n, dtype=torch.float64, device="cuda")
st = thread_state(x.device); ws = st.ws_ptr
c = config_struct(Q.ToleranceConfig(1e-8), Q.ExactBinning()); cr = ctypes.byref(c)
s = torch.cuda.current_stream().cuda_stream
for _ in range(6):
    lib.qdot_b200_begin(ws, s)
    lib.qdot_b200_pass1(x.data_ptr(), y.data_ptr(), n, 0, cr, n, ws, s)
    lib.qdot_b200_score_finalize(ws, n, cr, s)
    lib.qdot_b200_pass2_finalize(x.data_ptr(), y.data_ptr(), n, 0, ws, s)
torch.cuda.synchronize()
