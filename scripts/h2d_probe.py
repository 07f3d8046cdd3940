"""Host->device copy rate from pinned memory: one 2 GiB copy, chunked copies on
1 and 2 streams, and x+y on two streams (what e2e is bound by)."""
import time, torch
n = 1 << 28
x = torch.empty(n, dtype=torch.float64).pin_memory()
y = torch.empty(n, dtype=torch.float64).pin_memory()
x.fill_(1.0); y.fill_(2.0)
dx = torch.empty(n, dtype=torch.float64, device="cuda"); dy = torch.empty_like(dx)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def one(): dx.copy_(x, non_blocking=True); dy.copy_(y, non_blocking=True)
def two():
    with torch.cuda.stream(s1): dx.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2): dy.copy_(y, non_blocking=True)
def chunked(ch=1 << 24):
    for o in range(0, n, ch):
        st = s1 if (o // ch) % 2 == 0 else s2
        with torch.cuda.stream(st):
            dx[o:o + ch].copy_(x[o:o + ch], non_blocking=True); dy[o:o + ch].copy_(y[o:o + ch], non_blocking=True)
for name, f in (("serial x,y", one), ("two streams", two), ("chunked 16M x2 streams", chunked)):
    dt = t(f)
    print(f"{name}: {dt*1e3:.1f} ms  {2*n*8/dt/1e9:.1f} GB/s")
