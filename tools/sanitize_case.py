"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): C1 (640x480, 3 levels, 8x8 grid, k=4, 21x21) through every ABI
call and kernel variant — pyramid, dense and fused detection (with and without
mask / raw response), KLT (default, NCC-each-step, 11x11, guess + in_status,
track-list records), patches — plus 6 frames of the f1 keyframe tracker
(suppression mask, survival, Eq. 5, masked detection, refill).
usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2506_04359_b200 import vslam2d as v2d  # noqa: E402
from paper_2506_04359_b200.frontend import KeyframeTracker  # noqa: E402


def main():
    torch.cuda.set_device(0)
    W, H, L = 640, 480, 3
    f0, f1 = synth.shifted_pair(H, W, (3.2, -1.7), seed=1, pitch=640)
    d0 = torch.from_numpy(f0[None].copy()).cuda()
    d1 = torch.from_numpy(f1[None].copy()).cuda()
    p0, p1 = v2d.build_pyramid(d0, W, L), v2d.build_pyramid(d1, W, L)
    mask = torch.zeros_like(d0)
    mask[:, 100:200, 100:300] = 1
    for dense in (True, False):
        xy, sc, cnt, _ = v2d.detect_gftt(d0, W, 8, 8, k=4, border=11, dense=dense)
        v2d.detect_gftt(d0, W, 8, 8, k=4, border=11, dense=dense, want_resp=True, mask=mask)
        v2d.detect_gftt(d0, W, 4, 3, k=40, border=3, nms=0, dense=dense)
    pts = xy.view(1, -1, 2)
    rec = torch.zeros((1, pts.shape[1], 4), device="cuda")
    v2d.track_klt(d0, p0, d1, p1, W, L, pts, track_list=rec)
    v2d.track_klt(d0, p0, d1, p1, W, L, pts, flags=v2d.KLT_NCC_EACH_STEP)
    v2d.track_klt(d0, p0, d1, p1, W, L, pts, win=11)
    extra = torch.tensor([[[0.0, 0.0], [639.0, 479.0], [-1.0, -1.0], [5.5, 470.25]]],
                         device="cuda")
    guess = torch.full((1, 4, 2), 2.0, device="cuda")
    ins = torch.tensor([[0, 0, 0, 1]], dtype=torch.uint8, device="cuda")
    v2d.track_klt(d0, p0, d1, p1, W, L, extra, guess=guess, in_status=ins)
    v2d.extract_patches(d0, p0, W, L, pts, 9)
    # f1 keyframe tracker on a 2-camera 320x240 stream
    wl = synth.Workload("san", 12, 320, 240, 2, 3, grid_x=4, grid_y=3, k=6, motion=(7.0, 5.0),
                        stereo_disparity=0.0)
    st = synth.make_stream(wl, 7, "cuda")
    cfg = v2d.FrontendConfig(W=320, H=240, levels=3, grid_x=4, grid_y=3, k=6, border=11)
    kt = KeyframeTracker(cfg, 2, "cuda", wl.pitch, T=0.9, min_sep=8.0)
    ptr = lambda t: v2d.ptrs_of(st.frames[:, t])
    kt.start(ptr(0))
    for t in range(1, 7):
        kt.step(ptr(t), ptr(t - 1))
    torch.cuda.synchronize()
    print("sanitize case ok:", int((rec[..., 2] == 0).sum()), "tracked;",
          "keyframe flag", int(kt.flag.item()))


if __name__ == "__main__":
    main()
