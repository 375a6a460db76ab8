"""Probe: NMS candidates per grid cell on the bench workloads (input for the K2 pass B
design).  Runs detection through the C-ABI with a caller-owned
workspace and counts the pass-A map's candidates inside each cell's eligible region
(nms = 1: the half-resolution map, one int32 word per pixel pair, bits(R) | dx << 31 or
all ones; decoded back to a per-pixel candidate image here).  usage (GPU box): python tools/cand_density.py [c2 c3 c4 c5]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2506_04359_b200 import vslam2d as v  # noqa: E402

out = {}
for name in sys.argv[1:] or ["c2", "c3", "c4", "c5"]:
    wl = synth.WORKLOADS[name]
    st = synth.make_stream(wl, 2, device="cuda", cams=[0, min(1, wl.cams - 1)])
    fr = st.frames.reshape(-1, wl.H, wl.pitch).contiguous()
    B = fr.shape[0]
    kk = v.grid_k(wl.grid_x, wl.grid_y, wl.k, wl.K_min)
    xy = torch.empty((B, wl.grid_y, wl.grid_x, kk, 2), device="cuda")
    sc = torch.empty((B, wl.grid_y, wl.grid_x, kk), device="cuda")
    cnt = torch.empty((B, wl.grid_y * wl.grid_x), dtype=torch.int32, device="cuda")
    ws = torch.empty((B, wl.H, v.workspace_pitch(wl.W)), device="cuda")
    v.detect_gftt_ptrs(v.ptrs_of(fr), fr.stride(1), B, wl.W, wl.H, wl.grid_x, wl.grid_y, wl.k,
                       wl.K_min, 0.0, wl.border, 1, xy, sc, cnt, None, None, None, ws)
    torch.cuda.synchronize()
    wp = v.workspace_pitch(wl.W) // 2  # words per half-map row, rows packed from the start
    words = ws.view(torch.int32).reshape(-1)[: B * wl.H * wp].view(B, wl.H, wp)
    valid = words != -1
    dx = (words < 0) & valid  # bit 31 set on a candidate = right pixel of the pair
    c = torch.zeros((B, wl.H, 2 * words.shape[2]), dtype=torch.bool, device="cuda")
    c[:, :, 0::2] = valid & ~dx
    c[:, :, 1::2] = dx
    c = c[:, :, : wl.W]
    per = []
    for cy in range(wl.grid_y):
        y0 = max(cy * wl.H // wl.grid_y, wl.border)
        y1 = min((cy + 1) * wl.H // wl.grid_y, wl.H - wl.border)
        for cx in range(wl.grid_x):
            x0 = max(cx * wl.W // wl.grid_x, wl.border)
            x1 = min((cx + 1) * wl.W // wl.grid_x, wl.W - wl.border)
            per.append(c[:, y0:y1, x0:x1].sum(dim=(1, 2)))
    per = torch.stack(per, 1).float()
    px = (wl.W // wl.grid_x) * (wl.H // wl.grid_y)
    out[name] = {"cell_px": px, "k": kk, "cand_mean": per.mean().item(),
                 "cand_max": per.max().item(), "cand_min": per.min().item(),
                 "density": per.mean().item() / px}
    print(name, json.dumps(out[name]), flush=True)
