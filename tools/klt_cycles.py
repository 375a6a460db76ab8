"""Phase cycles of K3 from a V2D_KLT_CYC debug build (exp/lib_C.so): warp-elapsed SM
clocks per phase (template staging, template build, search staging, Gauss-Newton
steps, NCC gate) as shares of the whole-warp time, on one c5 (or given config) step.
Also prints the launch time of the instrumented build (compare with klt_win_probe on
the production build to see how much the clock reads distort).
usage: python tools/klt_cycles.py [config] [lib]   (on the GPU box)"""
import ctypes
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c5"
libname = sys.argv[2] if len(sys.argv) > 2 else "C"
shutil.copy(os.path.join(ROOT, "exp", f"lib_{libname}.so"),
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
cur, prev, parity = sched.tables(0)
fe.step(cur, prev, parity)
c = fe.cfg
pts = fe.kp_xy[:-1].reshape(fe.B, fe.P, 2).contiguous()
pos, stt, it = torch.empty_like(fe.pos), torch.empty_like(fe.status), torch.empty_like(fe.iters)
args = (prev, fe.prev_pyr_ptrs[parity], cur, fe.pyr_ptrs[parity], fe.pitch, fe.B, c.W, c.H,
        c.levels, pts, None, None, fe.P, c.win, c.iters, c.eps, c.ncc_min, c.min_eig, pos, stt,
        None, it)
lib = v2d.load()
cyc = (ctypes.c_ulonglong * 512)()
v2d.track_klt_ptrs(*args)
torch.cuda.synchronize()
lib.v2d_debug_klt_cycles(cyc, 1)
reps = 10
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    v2d.track_klt_ptrs(*args)
b.record()
torch.cuda.synchronize()
lib.v2d_debug_klt_cycles(cyc, 1)
ms = a.elapsed_time(b) / reps
tot = [sum(cyc[8 * s + i] for s in range(64)) for i in range(8)]
names = ["tmpl_stage", "tmpl_build", "search_stage", "gn_steps", "ncc"]
tot[3] -= tot[2]  # the first search staging happens inside the Gauss-Newton loop
whole = max(tot[5], 1)
nw = reps * fe.B * fe.P
print(f"{cfgname} lib_{libname}: {ms:.4f} ms per launch; whole-warp cycles per warp "
      f"{whole / nw:.0f}")
print("  " + "  ".join(f"{n} {100 * t / whole:.1f}%" for n, t in zip(names, tot)) +
      f"  other {100 * (whole - sum(tot[:5])) / whole:.1f}%")
