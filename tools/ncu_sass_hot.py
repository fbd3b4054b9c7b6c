"""Top stall-sampled SASS lines of one kernel in an ncu report (needs --import-source / lineinfo).
    python tools/ncu_sass_hot.py report.ncu-rep [N] [context]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for i, r in enumerate(rows[2:]):
    try:
        data.append((int(r[si]), i, r[1].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print("total samples", tot)
for v, i, src in sorted(data, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}% {i:5d} {src[:100]}")
