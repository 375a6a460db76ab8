"""KLT event counters of a V2D_KLT_STATS debug build (exp/lib_S.so) on the bench
data of a config: template paths, stagings, re-stagings, GN steps, eig skips.
usage: python tools/klt_stats.py [config]   (on the GPU box)"""
import ctypes
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c5"
shutil.copy(os.path.join(ROOT, "exp", "lib_S.so"),
            os.path.join(ROOT, "paper_2506_04359_b200", "libvslam2d.so"))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2506_04359_b200 import vslam2d as v2d  # noqa: E402
from paper_2506_04359_b200.frontend import RingSchedule  # noqa: E402

wl = synth.WORKLOADS[cfgname]
lay = bench.bench_layout(wl, 1)
st = synth.make_stream(wl, lay["R"], "cuda")
fe = bench.make_frontend(wl, lay["streams"], lay["F"], torch.device("cuda"))
sched = RingSchedule(st.frames, lay["F"])
fe.prime(sched.before_first, 1)
lib = v2d.load()
buf = (ctypes.c_ulonglong * 16)()
for s in range(3):
    lib.v2d_debug_klt_stats(buf, 1)
    cur, prev, parity = sched.tables(s)
    fe.step(cur, prev, parity)
    torch.cuda.synchronize()
lib.v2d_debug_klt_stats(buf, 1)
names = ["kp_levels_with_template", "interior_template", "border_template", "gn_steps",
         "search_stagings", "re_stagings", "eig_skips", "u8_stage_fast", "u8_stage_clamped",
         "f32_stage_fast", "f32_stage_clamped"]
n_kp = int((fe.status != 4).sum())
print(f"{cfgname}: attempted keypoints {n_kp}")
for i, n in enumerate(names):
    print(f"  {n:26s} {buf[i]:>10d}  per attempted kp {buf[i] / max(n_kp, 1):.3f}")
