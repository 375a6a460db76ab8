"""Time v2d_track_klt alone for a given window on the c5 bench data (B = 32 images,
2048 slots each), e.g. for ncu captures of one variant.
usage: python tools/klt_win_probe.py [win] [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2506_04359_b200 import vslam2d as v2d  # noqa: E402
from paper_2506_04359_b200.frontend import RingSchedule  # noqa: E402

win = int(sys.argv[1]) if len(sys.argv) > 1 else 11
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
levels_arg = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # track through fewer levels
wl = synth.WORKLOADS["c5"]
lay = bench.bench_layout(wl, 1)
st = synth.make_stream(wl, lay["R"], "cuda")
fe = bench.make_frontend(wl, lay["streams"], lay["F"], torch.device("cuda"))
sched = RingSchedule(st.frames, lay["F"])
fe.prime(sched.before_first, 1)
cur, prev, parity = sched.tables(0)
fe.step(cur, prev, parity)
c = fe.cfg
pts = fe.kp_xy[:-1].reshape(fe.B, fe.P, 2).contiguous()
pos = torch.empty_like(fe.pos)
stt = torch.empty_like(fe.status)
it = torch.empty_like(fe.iters)
args = (prev, fe.prev_pyr_ptrs[parity], cur, fe.pyr_ptrs[parity], fe.pitch, fe.B, c.W, c.H,
        levels_arg or c.levels, pts, None, None, fe.P, win, c.iters, c.eps, c.ncc_min, c.min_eig, pos, stt,
        None, it)
v2d.track_klt_ptrs(*args)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    v2d.track_klt_ptrs(*args)
b.record()
torch.cuda.synchronize()
print(f"win {win} levels {levels_arg or c.levels}: {a.elapsed_time(b) / reps:.4f} ms per launch, "
      f"steps/kp {float((it & 0xFFFFFF).sum()) / max(1, int((stt != 4).sum())):.2f}")
