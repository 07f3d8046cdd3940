"""Per-instruction stall hot spots of one kernel in an ncu report.

    python tools/sass_stalls.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
rows = rows[starts[0]:starts[1]]
hdr, data = rows[1], [r for r in rows[2:] if len(r) > 5]
iE = hdr.index("Instructions Executed")
iS = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iS] or 0) for r in data) or 1
print(f"{rows[0][1][:80]}: {len(data)} static, {sum(1 for r in data if int(r[iE] or 0))} executed, "
      f"{sum(int(r[iE] or 0) for r in data)} warp insts, {tot} samples")
for i in sorted(sorted(range(len(data)), key=lambda i: -int(data[i][iS] or 0))[:top]):
    r = data[i]
    print(f"  {i:5d} {int(r[iS]) / tot * 100:5.1f}% ex={r[iE]:>8} {r[1][:80]}")
