"""Turn the GPU-box captures of tools/gpu_profile_r02.sh (gpurun_out/) into the
committed summaries under profiles/ (run here, no GPU needed):
  {tag}_launches_{cfg}.csv / .txt   ncu launch list (gpu__time_duration, serialised)
  {tag}_full_{cfg}_{kernel}.txt     ncu --set full summaries (+ SASS opcode mix)
  traffic_{cfg}.json                DRAM bytes per launch per kernel (bench roofline)
usage: python tools/make_profiles.py [tag=r02] [cfg=c5]"""
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
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
cfg = sys.argv[2] if len(sys.argv) > 2 else "c5"
KERNELS = ("pyramid_kernel", "gftt_dense_kernel", "gftt_select", "klt_kernel")

# ---- launch list -----------------------------------------------------------
src = os.path.join(GO, f"{tag}_launches_{cfg}.csv")
shutil.copy(src, os.path.join(PR, f"{tag}_launches_{cfg}.csv"))
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
out_txt = os.path.join(PR, f"{tag}_launches_{cfg}.txt")
with open(out_txt, "w") as f:
    f.write("# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
    f.write(f"# command: python bench.py --config {cfg} --steps 3 --warmup 2 --no-e2e "
            f"--no-cpu-baseline   (bench launch configuration)\n")
    f.write("kernel, launches, mean_us, min_us, max_us\n")
    for k, v in ours.items():
        f.write(f"{k}, {len(v)}, {sum(v) / len(v):.1f}, {min(v):.1f}, {max(v):.1f}\n")
    f.write("# share of one step (sum of the kernel means): " + ", ".join(
        f"{k} {100 * sum(v) / len(v) / tot:.1f}%" for k, v in ours.items()) + "\n")
print(open(out_txt).read())

# ---- full captures ---------------------------------------------------------
summ = os.path.join(ROOT, "tools", "ncu_summary.py")
for k in KERNELS:
    rep = os.path.join(GO, f"{tag}_full_{cfg}_{k}.ncu-rep")
    if os.path.exists(rep):
        out = subprocess.run([sys.executable, summ, rep, "--ops"], capture_output=True,
                             text=True).stdout
        open(os.path.join(PR, f"{tag}_full_{cfg}_{k}.txt"), "w").write(out)


def dram_bytes(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(out.splitlines()))
    hh = rr[0]
    b = 0.0
    for r in rr[2:3]:
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v = r[hh.index(m)].replace(",", "")
            unit = rr[1][hh.index(m)]
            b += float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return b


tr = {}
for k, key in (("klt_kernel", "klt"), ("pyramid_kernel", "pyramid"),
               ("gftt_dense_kernel", "gftt_dense_kernel"),
               ("gftt_select", "gftt_select_kernel")):
    rep = os.path.join(GO, f"{tag}_full_{cfg}_{k}.ncu-rep")
    if os.path.exists(rep):
        tr[key] = dram_bytes(rep)
if "gftt_dense_kernel" in tr and "gftt_select_kernel" in tr:
    tr["gftt_topk"] = tr["gftt_dense_kernel"] + tr["gftt_select_kernel"]
tr["_source"] = (f"ncu --set full, one launch each ({cfg} bench launch configuration), "
                 f"dram__bytes_read.sum + dram__bytes_write.sum, bytes per launch; gftt_topk = "
                 f"gftt_dense + gftt_select; profiles/{tag}_full_{cfg}_*.txt")
json.dump(tr, open(os.path.join(PR, f"traffic_{cfg}.json"), "w"), indent=1)
print(json.dumps(tr, indent=1))
