"""Pass 1 vs the read probe (the same 4 GiB, same load pattern, no compute)
under identical sustained conditions: alternating blocks of back-to-back
launches, CUDA events per launch; reports the mean of each block."""
import ctypes, json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2105_00115_b200 as Q
from paper_2105_00115_b200 import _lib
from paper_2105_00115_b200.device import config_struct, thread_state

n = 1 << 28
lib = _lib.load()
rng = np.random.default_rng(0)
x = torch.from_numpy(rng.standard_normal(n)).cuda()
y = torch.from_numpy(rng.standard_normal(n)).cuda()
st = thread_state(x.device)
ws = st.ws_ptr
s = torch.cuda.current_stream().cuda_stream
c = config_struct(Q.ToleranceConfig(1e-8), Q.ExactBinning())
c.reserved = int(os.environ.get("P1MODE", "0"))      # pass-1 mode knob (qdot_b200_pass1), 0 = auto
out = torch.zeros(1, dtype=torch.float64, device="cuda")


def p1():
    lib.qdot_b200_begin(ws, s)
    lib.qdot_b200_pass1(x.data_ptr(), y.data_ptr(), n, 0, ctypes.byref(c), n, ws, s)


def probe():
    lib.qdot_b200_read_probe(x.data_ptr(), n, out.data_ptr(), s)
    lib.qdot_b200_read_probe(y.data_ptr(), n, out.data_ptr(), s)


def block(fn, reps=100):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return statistics.mean(a.elapsed_time(b) for a, b in ev)


for _ in range(3):
    p1(); probe()
torch.cuda.synchronize()
rows = []
for r in range(int(os.environ.get("BLOCKS", "6"))):
    rows.append({"block": r, "pass1_ms": block(p1), "probe_ms": block(probe)})
    print(json.dumps(rows[-1]), flush=True)
p = statistics.mean(r["pass1_ms"] for r in rows)
q = statistics.mean(r["probe_ms"] for r in rows)
print(json.dumps({"pass1_ms": p, "probe_ms": q, "pass1_over_probe": p / q,
                  "pass1_GBps": n * 16 / p / 1e6, "probe_GBps": n * 16 / q / 1e6}))
