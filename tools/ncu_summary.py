"""Summarise ncu captures for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py gpurun_out/pass1_X.ncu-rep profiles/r1_pass1 [--n 268435456]
    python tools/ncu_summary.py --launches gpurun_out/launches.csv profiles/r1_launches

Writes <out>.txt (human readable: speed-of-light, memory, stalls, top SASS
lines) and <out>.json (the numbers bench.py reads: dram bytes per launch).
"""

import argparse
import csv
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("dram__bytes.sum.per_second", "dram bandwidth"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def to_bytes(val, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(val.replace(",", "")) * mult.get(unit, 1)


def summarise(rep, out, n):
    h, u, rows = raw(rep)
    txt = []
    js = {"report": rep, "n": n, "kernels": []}
    for row in rows:
        name = row[h.index("Kernel Name")]
        d = dict(zip(h, row))
        units = dict(zip(h, u))
        txt.append(f"== {name}")
        kj = {"kernel": name}
        for key, label in KEYS:
            if key in d:
                txt.append(f"  {label:34s} {d[key]:>18s} {units[key]}")
                kj[key] = d[key] + " " + units[key]
        stalls = []
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                if v > 0.05:
                    stalls.append((v, k.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
        txt.append("  stalls (warps per issue): " + ", ".join(f"{s}={v:.2f}" for v, s in sorted(stalls, reverse=True)))
        rd = to_bytes(d["dram__bytes_read.sum"], units["dram__bytes_read.sum"])
        wr = to_bytes(d["dram__bytes_write.sum"], units["dram__bytes_write.sum"])
        kj["dram_bytes_per_launch"] = rd + wr
        js["kernels"].append(kj)
    if js["kernels"]:
        js["dram_bytes_per_launch"] = js["kernels"][0]["dram_bytes_per_launch"]
    # top SASS lines by stall samples
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(src.splitlines()))
    if len(srows) > 2:
        hh = srows[1]
        try:
            si, ai, ti, ei = (hh.index("Source"), hh.index("Address"),
                              hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed"))
            data = []
            for r in srows[2:]:
                try:
                    data.append((int(r[ti] or 0), r[ai][-5:], r[ei], r[si][:70]))
                except (ValueError, IndexError):
                    pass
            tot = sum(x[0] for x in data) or 1
            txt.append("  top SASS by stall samples:")
            for x in sorted(data, reverse=True)[:12]:
                txt.append(f"    {100 * x[0] / tot:5.1f}%  {x[1]}  exec={x[2]:>9s}  {x[3]}")
        except ValueError:
            pass
    with open(out + ".txt", "w") as f:
        f.write("\n".join(txt) + "\n")
    with open(out + ".json", "w") as f:
        json.dump(js, f, indent=1)
    print("\n".join(txt))


def launches(csvfile, out):
    rows = list(csv.reader(open(csvfile)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = {}
    seq = []
    for r in rows[i + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        us = v / 1000.0 if r[ui] == "ns" else (v * 1000.0 if r[ui] == "ms" else v)
        seq.append((name, us))
        per.setdefault(name, []).append(us)
    tot = sum(us for _, us in seq) or 1
    lines = ["launch list (ncu gpu__time_duration, cold-cache and serialised: compare shares)",
             f"{'kernel':60s} {'launches':>8s} {'mean us':>10s} {'share':>7s}"]
    js = {"csv": csvfile, "kernels": {}}
    for name, v in sorted(per.items(), key=lambda t: -sum(t[1])):
        lines.append(f"{name[:60]:60s} {len(v):8d} {sum(v) / len(v):10.2f} {100 * sum(v) / tot:6.1f}%")
        js["kernels"][name] = {"launches": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / tot}
    lines.append("sequence:")
    lines += [f"  {n[:60]:60s} {us:10.2f} us" for n, us in seq]
    with open(out + ".txt", "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(out + ".json", "w") as f:
        json.dump(js, f, indent=1)
    print("\n".join(lines[:12]))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("out")
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--launches", action="store_true")
    a = ap.parse_args()
    if a.launches:
        launches(a.src, a.out)
    else:
        summarise(a.src, a.out, a.n)
    sys.exit(0)
