"""Summarise an ncu report's SASS page: instruction mix, per-iteration frequency buckets, stall reasons.

    python tools/sass_hist.py report.ncu-rep [iters]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
iters = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
iE = hdr.index("Instructions Executed")
iS = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iE] or 0) for r in data)
ts = sum(int(r[iS] or 0) for r in data) or 1
print(f"warp instructions {tot}  samples {ts}")
c, s = Counter(), Counter()
for r in data:
    parts = r[1].split()
    if not parts:
        continue
    m = parts[1] if parts[0].startswith("@") else parts[0]
    m = m.split(".")[0]
    c[m] += int(r[iE] or 0)
    s[m] += int(r[iS] or 0)
for m, v in c.most_common(20):
    print(f"  {m:10s} {v / tot * 100:5.1f}% inst  {s[m] / ts * 100:5.1f}% stall samples")
if iters:
    b = Counter()
    for r in data:
        e = int(r[iE] or 0)
        if e:
            b[round(e / iters, 2)] += e
    print("per-iteration multiplicity buckets:")
    for k, v in sorted(((k, v) for k, v in b.items() if k > 0), key=lambda kv: -kv[1])[:12]:
        print(f"  x{k:7.3f}: {v / tot * 100:5.1f}% of instructions, {v / (k * iters):.0f} static instrs")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, v = rr[0], rr[2]
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(x) for k, x in zip(h, v)
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k and x.replace(".", "").isdigit()}
tot_st = sum(st.values()) or 1
print("stall reasons:", ", ".join(f"{k} {x / tot_st * 100:.0f}%" for k, x in sorted(st.items(), key=lambda kv: -kv[1])[:8]))
for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed"):
    if k in h:
        print(f"{k} = {v[h.index(k)]} {rr[1][h.index(k)]}")
