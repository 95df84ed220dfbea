#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel
totals and shares, and (optionally) one `ncu --set full` report's key counters.

    python scripts/ncu_summary.py launches.csv [--full report.ncu-rep ...] > profiles/rNN_summary.md
"""
import collections
import csv
import re
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [r for r in rows if r and r[0] == "ID"][0]
    data = [dict(zip(hdr, r)) for r in rows if r and r[0] != "ID" and len(r) == len(hdr)]
    agg = collections.OrderedDict()
    for d in data:
        name = re.sub(r"\(.*", "", d["Kernel Name"])
        name = name.replace("ssm::<unnamed>::", "").replace("void ", "")
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[d["Metric Unit"]]
        key = (name[:70], d["Grid Size"])
        a = agg.setdefault(key, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"]) * scale
    ours = {k: v for k, v in agg.items() if not k[0].startswith("at::") and "at::" not in k[0][:20]}
    tot = sum(v[1] for v in ours.values())
    print(f"### Launch list `{path}` (our kernels only; cold-cache, serialised)\n")
    print("| kernel | grid | launches | total µs | avg µs | share |")
    print("|---|---|---|---|---|---|")
    for (k, g), (n, t) in sorted(ours.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {g} | {n} | {t:.1f} | {t / n:.2f} | {100 * t / tot:.1f}% |")
    print()


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "Kernel Name", "Grid Size", "Block Size"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    print(f"### Full report `{path}`\n")
    for v in rows[2:]:
        print("| metric | value | unit |\n|---|---|---|")
        for i, name in enumerate(h):
            if name in KEYS:
                val = v[i] if name != "Kernel Name" else re.sub(r"\(.*", "", v[i])[:80]
                print(f"| {name} | {val} | {u[i]} |")
        print()


if __name__ == "__main__":
    args = sys.argv[1:]
    i = 0
    while i < len(args):
        if args[i] == "--full":
            i += 1
            while i < len(args) and args[i].endswith(".ncu-rep"):
                full(args[i])
                i += 1
        else:
            launches(args[i])
            i += 1
