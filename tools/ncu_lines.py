"""Aggregate an ncu report's SASS metrics by CUDA source line (needs -lineinfo).
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
inst, stall, src = collections.Counter(), collections.Counter(), {}
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        ln = int(r[0])
    except ValueError:
        continue
    src[ln] = r[1][:90]
    ie = hdr.index("Instructions Executed")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        inst[ln] += int(r[ie] or 0)
        stall[ln] += int(r[ist] or 0)
    except ValueError:
        pass
ti, ts = sum(inst.values()), sum(stall.values())
print(f"total inst {ti}  stall samples {ts}")
for ln, n in sorted(inst.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{ln:5d} {100 * n / ti:5.1f}% inst {100 * stall[ln] / max(ts, 1):5.1f}% stall | {src.get(ln, '').strip()}")
