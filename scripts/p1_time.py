"""Time pass 1 alone (CUDA events) at n = 2^28 for the current pass-1 variant.
Usage: QDOT_B200_P1_VARIANT=k python scripts/p1_time.py [--norm] [--mode 0|1|2] [--data normal|illcond]"""
import argparse, ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2105_00115_b200 as Q
from paper_2105_00115_b200 import _lib
from paper_2105_00115_b200.device import config_struct, thread_state

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 28)
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--data", default="normal")
ap.add_argument("--eps", type=float, default=1e-8)
ap.add_argument("--norm", action="store_true")
args = ap.parse_args()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
if args.data == "normal":
    x = torch.randn(args.n, dtype=torch.float64, device=dev, generator=g)
    y = torch.randn(args.n, dtype=torch.float64, device=dev, generator=g)
else:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.oracle import gen_illcond
    xh, yh = gen_illcond(args.n, seed=0)
    x = torch.from_numpy(xh).to(dev); y = torch.from_numpy(yh).to(dev)
if args.norm:
    y = x
nm = 1 if args.norm else 0
lib = _lib.load()
st = thread_state(dev)
c = config_struct(Q.ToleranceConfig(args.eps), Q.ExactBinning())
c.reserved = args.mode
s = torch.cuda.current_stream().cuda_stream
ws = st.ws_ptr
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
for i in range(3 + args.reps):
    if i >= 3: sev[i - 3][0].record()
    _lib.check(lib.qdot_b200_begin(ws, s))
    if i >= 3: evs[i - 3][0].record()
    _lib.check(lib.qdot_b200_pass1(x.data_ptr(), y.data_ptr(), args.n, nm, ctypes.byref(c), args.n, ws, s))
    if i >= 3: evs[i - 3][1].record()
    _lib.check(lib.qdot_b200_score(ws, args.n, ctypes.byref(c), s))
    _lib.check(lib.qdot_b200_pass2(x.data_ptr(), y.data_ptr(), args.n, nm, ws, s))
    _lib.check(lib.qdot_b200_finalize(ws, s))
    if i >= 3: sev[i - 3][1].record()
_lib.check(lib.qdot_b200_fetch(ws, ctypes.byref(st.result), st.bins, 4196, s))
torch.cuda.synchronize()
ts = sorted(a.elapsed_time(b) for a, b in evs)
med = ts[len(ts) // 2]
ss = sorted(a.elapsed_time(b) for a, b in sev)
print(json.dumps({"variant": os.environ.get("QDOT_B200_P1_VARIANT", "0"), "mode": args.mode, "data": args.data,
                  "pass1_ms_median": med, "pass1_ms_min": ts[0], "norm": args.norm, "GBps": args.n * (8 if args.norm else 16) / med / 1e6,
                  "step_ms_median": ss[len(ss) // 2], "value": st.result.value, "p2": st.result.pass2_needed}))
