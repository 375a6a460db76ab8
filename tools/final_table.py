"""Print the results-table rows from the bench lines of tools/gpu_final_r02.sh
(gpurun_out/{tag}_bench_*.log) as markdown, for DESIGN.md §10 / README / BASELINE.md §4.
usage: python tools/final_table.py [tag=r02k]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02k"


def line(name):
    p = os.path.join(ROOT, "gpurun_out", f"{tag}_bench_{name}.log")
    for ln in reversed(open(p).read().splitlines()):
        if ln.startswith("{"):
            return json.loads(ln)
    raise SystemExit(f"no JSON line in {p}")


for name in ("c1", "c2", "c3", "c4", "default"):
    d = line(name)
    k = d["kernels"]
    r = d["rooflines_all_kernels"]
    ms = " / ".join(f"{k[n]['ms_per_launch']:.3f}" for n in ("pyramid", "gftt_topk", "klt"))
    print(f"| {name} | {d['value']:,.0f} | {d['keypoints_tracked_per_s'] / 1e6:.1f} M | "
          f"{d['e2e']['value']:,.0f} | {d['ms_per_step']:.3f} | {ms} | "
          f"{100 * r['pyramid']['frac']:.1f} | {100 * d['hbm_full_path']['frac_of_measured']:.1f} | "
          f"{100 * r['klt']['frac']:.1f} | {100 * r['gftt_topk']['frac']:.1f} | "
          f"{d['cpu_baseline']['value']:.2f} | clocks {d['clocks']['sm_mhz']:.0f} "
          f"{d['clocks']['reasons']} |")
