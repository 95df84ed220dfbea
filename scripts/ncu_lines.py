"""Warp-stall samples of an ncu report per CUDA source line (ncu --page source --print-source
cuda,sass), with each line's dominant stall reasons.

    python scripts/ncu_lines.py report.ncu-rep [top]
"""
import csv
import collections
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = "?"
hdr = None
lines = []
total = 0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or r[2] != "-" or not r[0]:
        continue   # SASS rows (the CUDA line rows carry the per-line aggregate)
    try:
        n = int(r[4] or 0)
    except ValueError:
        continue
    rs = collections.Counter()
    for i, k in enumerate(hdr):
        if k.startswith("stall_") and "Not Issued" not in k and i < len(r):
            try:
                rs[k[6:]] += int(r[i] or 0)
            except ValueError:
                pass
    total += n
    lines.append((n, f"{fname}:{r[0]}", r[1].strip()[:100], rs))
print(f"total samples {total}")
for n, loc, src, rs in sorted(lines, key=lambda x: -x[0])[:top]:
    why = ", ".join(f"{k} {v}" for k, v in rs.most_common(3) if v)
    print(f"{n:7d} {100 * n / max(total, 1):5.1f}%  {loc:22s} {src}   [{why}]")
