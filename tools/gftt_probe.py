"""Time v2d_detect_gftt (K2: pass A + pass B) alone on the bench data of a config
(B = 32 camera-frames); run under ncu for the per-pass split.
usage: python tools/gftt_probe.py [config] [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2506_04359_b200 import vslam2d as v2d  # noqa: E402
from paper_2506_04359_b200.frontend import RingSchedule  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
wl = synth.WORKLOADS[cfgname]
lay = bench.bench_layout(wl, 1)
st = synth.make_stream(wl, lay["R"], "cuda")
fe = bench.make_frontend(wl, lay["streams"], lay["F"], torch.device("cuda"))
sched = RingSchedule(st.frames, lay["F"])
fe.prime(sched.before_first, 1)
cur, prev, parity = sched.tables(0)
c = fe.cfg
args = (cur, fe.pitch, fe.B, c.W, c.H, c.grid_x, c.grid_y, c.k, c.K_min, c.min_score, c.border,
        c.nms, fe.kp_xy[1:], fe.kp_score[1:], fe.cell_count[1:])
v2d.detect_gftt_ptrs(*args, workspace=fe.ws)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    v2d.detect_gftt_ptrs(*args, workspace=fe.ws)
b.record()
torch.cuda.synchronize()
print(f"{cfgname}: detect {a.elapsed_time(b) / reps:.4f} ms per launch")
