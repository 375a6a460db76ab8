"""Turn the GPU-box captures of tools/gpu_profile_round.sh (gpurun_out/) into the
committed summaries under profiles/ (run here, no GPU needed):
  r01_launches_c2.csv / .txt   ncu launch list (gpu__time_duration, serialised)
  r01_full_c2_{klt,gftt,pyramid}.txt, r01_full_c5.txt   ncu --set full summaries
  traffic_c2.json              DRAM bytes per launch per kernel (bench roofline)
usage: python tools/make_profiles.py [tag=r01]"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GO = os.path.join(ROOT, "gpurun_out")
PR = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

# ---- launch list -----------------------------------------------------------
src = os.path.join(GO, "launches_c2.csv")
shutil.copy(src, os.path.join(PR, f"{tag}_launches_c2.csv"))
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > vi:
        n = r[ki].split("(")[0].split("::")[-1].split("<")[0]
        d.setdefault(n, []).append(float(r[vi].replace(",", "")) / 1e3)
ours = {k: v for k, v in d.items() if k.startswith(("pyramid", "gftt", "klt"))}
tot = sum(sum(v) / len(v) for v in ours.values())
with open(os.path.join(PR, f"{tag}_launches_c2.txt"), "w") as f:
    f.write("# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
    f.write("# command: python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline   "
            "(config c2, B=32 camera-frames/launch)\n")
    f.write("kernel, launches, mean_us, min_us, max_us\n")
    for k, v in ours.items():
        f.write(f"{k}, {len(v)}, {sum(v) / len(v):.1f}, {min(v):.1f}, {max(v):.1f}\n")
    f.write("# share of one step (sum of the kernel means): " + ", ".join(
        f"{k} {100 * sum(v) / len(v) / tot:.1f}%" for k, v in ours.items()) + "\n")
print(open(os.path.join(PR, f"{tag}_launches_c2.txt")).read())

# ---- full captures ---------------------------------------------------------
summ = os.path.join(ROOT, "tools", "ncu_summary.py")
for name in ("full_c2_klt", "full_c2_gftt", "full_c2_pyramid", "full_c5"):
    rep = os.path.join(GO, name + ".ncu-rep")
    if os.path.exists(rep):
        out = subprocess.run([sys.executable, summ, rep], capture_output=True, text=True).stdout
        open(os.path.join(PR, f"{tag}_{name}.txt"), "w").write(out)


def dram_bytes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(out.splitlines()))
    hh = rr[0]
    res = collections.OrderedDict()
    for r in rr[2:]:
        k = r[hh.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0]
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v = r[hh.index(m)].replace(",", "")
            unit = rr[1][hh.index(m)]
            b += float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        res[k] = b
    return res


tr = {}
for name, key in (("full_c2_klt", "klt"), ("full_c2_pyramid", "pyramid"), ("full_c2_gftt", None)):
    rep = os.path.join(GO, name + ".ncu-rep")
    if not os.path.exists(rep):
        continue
    for k, b in dram_bytes(rep).items():
        if key:
            tr[key] = b
        else:
            tr["gftt_topk"] = tr.get("gftt_topk", 0.0) + b
            tr[k] = b
tr["_source"] = ("ncu --set full, one launch each (B=32 c2 camera-frames), dram__bytes_read.sum + "
                 "dram__bytes_write.sum, bytes per launch; gftt_topk = gftt_dense + gftt_select; "
                 f"profiles/{tag}_full_c2_*.txt")
json.dump(tr, open(os.path.join(PR, "traffic_c2.json"), "w"), indent=1)
print(json.dumps(tr, indent=1))
