"""Small-n latency of one qdot (the solver regime): wall time
per call through qdot(), through run_device (no report), and the device time
of the pipeline (CUDA events), for n = 1e3 .. 1e7."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2105_00115_b200 as Q
from paper_2105_00115_b200.kernel import run_device
dev = torch.device("cuda", 0)
cfg = Q.ToleranceConfig(1e-8, Q.SplitMode.PER_BIN)
strat = Q.ExactBinning()
out = []
for n in [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1000", "10000", "100000", "1000000", "10000000"])]:
    g = torch.Generator(device=dev).manual_seed(1)
    x = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
    y = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
    for _ in range(20):
        Q.qdot(x, y, cfg)
    reps = 200
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): Q.qdot(x, y, cfg)
    t_api = (time.perf_counter() - t0) / reps
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): run_device(x, y, n, False, cfg, strat, timing=False)
    t_dev = (time.perf_counter() - t0) / reps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): run_device(x, y, n, False, cfg, strat, timing=False)
    e1.record(); torch.cuda.synchronize()
    out.append({"n": n, "qdot_api_us": t_api * 1e6, "run_device_us": t_dev * 1e6,
                "events_us_per_call": e0.elapsed_time(e1) / reps * 1e3})
    print(json.dumps(out[-1]), flush=True)
