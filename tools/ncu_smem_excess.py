"""Top SASS lines by excess shared-memory wavefronts (bank conflicts) in an ncu
report, with the CUDA source line each maps to (needs -lineinfo + --import-source).
usage: python tools/ncu_smem_excess.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ix = {n: h.index(n) for n in ("Address", "Source", "Instructions Executed", "L1 Wavefronts Shared",
                               "L1 Wavefronts Shared Ideal", "L1 Wavefronts Shared Excessive")}
tot = {"wf": 0, "ideal": 0, "exc": 0}
lines = []
for r in rows[2:]:
    if len(r) <= max(ix.values()):
        continue
    f = lambda k: int(float(r[ix[k]] or 0))
    wf, ide, exc = f("L1 Wavefronts Shared"), f("L1 Wavefronts Shared Ideal"), f("L1 Wavefronts Shared Excessive")
    tot["wf"] += wf
    tot["ideal"] += ide
    tot["exc"] += exc
    if exc:
        lines.append((exc, r[ix["Address"]], r[ix["Source"]][:60], f("Instructions Executed"), wf, ide))
print(f"shared wavefronts {tot['wf']}, ideal {tot['ideal']}, excessive {tot['exc']}")
for e in sorted(lines, reverse=True)[:top]:
    print(f"  excess {e[0]:>10}  {e[1]}  {e[2]:60s} inst {e[3]} wf {e[4]} ideal {e[5]}")
