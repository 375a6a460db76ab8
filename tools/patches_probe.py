"""Time / profile the f4 patches kernel alone on the c5 bench data (32 images,
65536 keypoints, 5 levels, 9x9).  usage: python tools/patches_probe.py [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2506_04359_b200 import vslam2d as v2d  # noqa: E402

wl = synth.WORKLOADS["c5"]
st = synth.make_stream(wl, 2, "cuda")
fr = st.frames[:, 0].contiguous()  # [32, H, pitch]
W, L = wl.W, wl.levels
pyr = v2d.build_pyramid(fr, W, L)
xy, sc, cnt, _ = v2d.detect_gftt(fr, W, 8, 8, K_min=2000, border=11)
pts = xy.view(fr.shape[0], -1, 2).contiguous()
out = v2d.extract_patches(fr, pyr, W, L, pts, 9)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
fp, pp = v2d.ptrs_of(fr), v2d.ptrs_of(pyr)  # pointer tables built once (host H2D copy)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    v2d.extract_patches_ptrs(fp, pp, fr.stride(1), fr.shape[0], W,
                             wl.H, L, pts, pts.shape[1], 9, out)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
print(f"patches c5: {ms:.4f} ms, {out.numel() * 4 / ms / 1e6:.1f} GB/s written")
