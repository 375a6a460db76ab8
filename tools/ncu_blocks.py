"""Dynamic instruction counts per straight-line SASS block of the profiled
kernel (run-length of equal execution counts) — shows where a kernel's
instructions go.  usage: python tools/ncu_blocks.py report.ncu-rep [min_pct]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc, ie = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
ist = h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[ia], 16), int(r[ie] or 0), int(r[ist] or 0), r[isrc].strip())
        for r in rows[2:] if len(r) > ie and r[ia].startswith("0x")]
base = data[0][0]
tot = sum(d[1] for d in data)
tots = sum(d[2] for d in data)
blocks, cur = [], None
for ad, n, st, src in data:
    if cur and n == cur[2]:
        cur[1] = ad
        cur[3] += 1
        cur[5] += st
    else:
        if cur:
            blocks.append(cur)
        cur = [ad, ad, n, 1, src, st]
blocks.append(cur)
print(f"total {tot} warp-instructions, {len(data)} static")
for b0, b1, n, cnt, src, st in blocks:
    if n * cnt > thr / 100 * tot:
        print(f"{b0 - base:05x}-{b1 - base:05x} x{cnt:4d} execs {n:>9d} = {100 * n * cnt / tot:5.1f}% "
              f"inst {100 * st / max(tots, 1):5.1f}% stall | {src[:60]}")
