"""C4 shape (65536 x 4096, eps 1e-6) per strategy: kernel time (CUDA events,
C ABI) and the qdot_batched() call (incl. the host reruns of flagged rows)."""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_00115_b200 as Q
from paper_2105_00115_b200 import _lib
from paper_2105_00115_b200.device import config_struct
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
R, L = 65536, 4096
X = torch.randn(R, L, dtype=torch.float64, device=dev, generator=g)
Y = torch.randn(R, L, dtype=torch.float64, device=dev, generator=g)
lib = _lib.load()
v = torch.empty(R, dtype=torch.float64, device=dev)
cn = torch.empty((R, 4), dtype=torch.int64, device=dev)
inf = torch.empty((R, 4), dtype=torch.int32, device=dev)
s = torch.cuda.current_stream().cuda_stream
for strat in sys.argv[1:] or ["exact", "ranged:3", "ranged:8", "split:3", "split:8"]:
    c = config_struct(Q.ToleranceConfig(1e-6), Q.parse_strategy(strat))
    def run():
        _lib.check(lib.qdot_b200_batched(X.data_ptr(), Y.data_ptr(), R, L, L, 0, ctypes.byref(c), v.data_ptr(),
                                         cn.data_ptr(), inf.data_ptr(), s))
    for _ in range(3): run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10): run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    flagged = int(((inf[:, 3] & (8 | 32)) != 0).sum())
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rep = Q.qdot_batched(X, Y, Q.ToleranceConfig(1e-6), strategy=Q.parse_strategy(strat))
    api_ms = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"strategy": strat, "kernel_ms": ms, "GBps": R * L * 16 / ms / 1e6, "flagged_rows": flagged,
                      "api_ms": api_ms, "rerun_rows": int(len(rep.general_rows))}), flush=True)
