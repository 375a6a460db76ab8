"""Top CUDA source lines by warp-stall samples with their dominant stall reasons
(SASS metrics attributed to source lines; needs -lineinfo + --import-source).
usage: python tools/ncu_stall_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
stall, reasons, src = collections.Counter(), collections.defaultdict(collections.Counter), {}
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    src[ln] = r[1][:70]
    d = dict(zip(hdr, r))
    try:
        stall[ln] += int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        pass
    for k, v in d.items():
        if k.startswith("stall_") and v:
            try:
                reasons[ln][k[6:]] += int(v)
            except ValueError:
                pass
tot = sum(stall.values())
print(f"stall samples {tot}")
for ln, n in stall.most_common(top):
    rs = ", ".join(f"{k} {v}" for k, v in reasons[ln].most_common(3))
    print(f"{ln:5d} {100 * n / max(tot, 1):5.1f}%  {src.get(ln, '').strip():70s} | {rs}")
