"""KLT cost model probe (GPU): time v2d_track_klt on c2-like data while varying
the iteration cap, the window and the level count; prints ms per launch and
the executed levels/steps so time ~ a*levels + b*steps can be fitted.
usage: python tools/klt_probe.py [config]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2506_04359_b200 import vslam2d as v  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = synth.WORKLOADS[cfg]
dev = torch.device("cuda")
st = synth.make_stream(wl, 2, device=dev)  # frames [C, 2, H, pitch] u8
C = st.frames.shape[0]
reps = max(1, 32 // C)
prev = st.frames[:, 0].repeat(reps, 1, 1).contiguous()
nxt = st.frames[:, 1].repeat(reps, 1, 1).contiguous()
B = prev.shape[0]


def run(levels, win, iters, flags=0, n=20):
    pp = v.build_pyramid(prev, wl.W, levels)
    pn = v.build_pyramid(nxt, wl.W, levels)
    kp, sc, cnt, _ = v.detect_gftt(prev, wl.W, wl.grid_x, wl.grid_y, wl.k, wl.K_min,
                                   border=(win - 1) // 2 + 1)
    pts = kp.reshape(B, -1, 2).contiguous()
    args = dict(win=win, iters=iters, eps=wl.eps, ncc_min=wl.ncc_min, min_eig=wl.min_eig,
                flags=flags)
    out = v.track_klt(prev, pp, nxt, pn, wl.W, levels, pts, **args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        out = v.track_klt(prev, pp, nxt, pn, wl.W, levels, pts, **args)
    e1.record()
    torch.cuda.synchronize()
    it = out[3].cpu().numpy().astype(np.int64)
    steps = int((it & 0xFFFFFF).sum())
    lv = int((it >> 24).sum())
    live = int((out[1].cpu().numpy() == 0).sum())
    ms = e0.elapsed_time(e1) / n
    print(f"L={levels} win={win:2d} iters={iters:2d} flags={flags} ms={ms:.4f} "
          f"kpts={pts.shape[0]*pts.shape[1]} levels={lv} steps={steps} tracked={live} "
          f"us/1k-level={ms*1e6/max(lv,1):.2f}", flush=True)


for iters in (1, 2, 3, 5, 10):
    run(wl.levels, wl.win, iters)
for win in (5, 11, 15, 21):
    run(wl.levels, win, wl.iters)
for L in (1, 2, 3, 4):
    run(L, wl.win, wl.iters)
