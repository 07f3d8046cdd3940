"""Phase clocks of the one-launch cluster path (CTA 0, SM cycles since entry,
written to A[A_SMALL + 1 .. + 7] by k_small): sample, stream, flush, cluster
barrier, merge + decision, score, exit."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2105_00115_b200 as Q
from paper_2105_00115_b200 import _lib
from paper_2105_00115_b200.device import config_struct, thread_state

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
lib = _lib.load()
x = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.randn(n, dtype=torch.float64, device="cuda")
st = thread_state(x.device)
c = config_struct(Q.ToleranceConfig(1e-8), Q.ExactBinning())
s = torch.cuda.current_stream().cuda_stream
out = torch.empty(8, dtype=torch.int64)
rows = []
try:
    from cuda.bindings import runtime as cudart          # cuda-python >= 12.8
except ImportError:
    from cuda import cudart
for i in range(30):
    lib.qdot_b200_enqueue(x.data_ptr(), y.data_ptr(), n, 0, ctypes.byref(c), st.ws_ptr, s)
    torch.cuda.synchronize()
    cudart.cudaMemcpy(out.data_ptr(), st.ws_ptr + 12664 * 8, 64, cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    rows.append(out.numpy().copy())
a = np.array(rows[5:])
print(json.dumps({"n": n, "small_state": int(a[-1][0]),
                  "phase_cycles_median": [int(v) for v in np.median(a[:, 1:], axis=0)]}))
