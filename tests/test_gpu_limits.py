"""Edge and limit cases of the C ABI on the GPU (task ③: empty inputs, maximum sizes).

* Empty batches: every call with B = 0 (and KLT / patches with P = 0) returns V2D_OK and
  leaves its outputs untouched (canary-filled).
* Maximum sizes in one run, compared with the oracle: a 3840x2160 frame with the maximum
  8 pyramid levels (every level bit-exact), detection on a 16x16 grid with the maximum
  k = 256 (bit-exact), and KLT with the largest window (29x29) through all 8 levels on a
  sample of the detected keypoints (oracle parity bands)."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle.parity import POS_TOL, compare_klt

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2506_04359_b200 import vslam2d as v2d


def _canary(shape, dtype):
    t = torch.full(shape, 7, dtype=dtype, device="cuda")
    return t, t.clone()


def test_empty_batches_are_noops():
    L = v2d.load()
    N = None
    st = torch.cuda.current_stream().cuda_stream
    out, ref = _canary((64,), torch.float32)
    p = ctypes.c_void_p(out.data_ptr())
    f = ctypes.c_float
    # B = 0 everywhere (null inputs are allowed when there is nothing to read)
    assert L.v2d_build_pyramid(N, 64, 0, 64, 64, 3, N, st) == 0
    assert L.v2d_detect_gftt(N, 64, 0, 64, 64, 2, 2, 4, 0, f(0.0), 3, 1, p, p, p, N, N, N, N,
                             st) == 0
    assert L.v2d_track_klt(N, N, N, N, 64, 0, 64, 64, 3, N, N, N, 16, 21, 10, f(0.01), f(0.8),
                           f(0.01), p, p, N, N, N, 0, st) == 0
    assert L.v2d_extract_patches(N, N, 64, 0, 64, 64, 3, N, 16, 9, p, st) == 0
    assert L.v2d_track_survival(N, N, 0, 16, p, st) == 0
    assert L.v2d_refill_tracks(p, p, 2, 2, 4, p, 0, 16, p, p, p, p, p, st) == 0
    # P = 0 with a real batch: nothing to track or sample
    fr = torch.zeros((2, 64, 64), dtype=torch.uint8, device="cuda")
    pyr = v2d.build_pyramid(fr, 64, 3)
    pts = torch.empty((2, 0, 2), device="cuda")
    pos, stt, ncc, it = v2d.track_klt(fr, pyr, fr, pyr, 64, 3, pts)
    assert pos.numel() == 0 and stt.numel() == 0
    assert v2d.extract_patches(fr, pyr, 64, 3, pts).numel() == 0
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_maximum_sizes_4k_8_levels_k256_win29():
    W, H, levels, gx, gy, k, win = 3840, 2160, 8, 16, 16, 256, 29
    wl = synth.Workload("mx", 14, W, H, 1, levels, motion=(2.5, -1.5), stereo_disparity=0.0)
    st = synth.make_stream(wl, 2, "cpu")
    fr = st.frames[0, :, :, :W].numpy().copy()          # [2, H, W]
    pitch = synth.round_up(W, 64)
    dev = torch.zeros((2, H, pitch), dtype=torch.uint8)
    dev[:, :, :W] = torch.from_numpy(fr)
    dev = dev.cuda()
    # pyramid: every level bit-exact
    pyr = v2d.build_pyramid(dev, W, levels)
    lay = v2d.pyramid_layout(W, H, levels)
    planes0, dense0 = oracle.build_pyramid(fr[0], levels)
    planes1, dense1 = oracle.build_pyramid(fr[1], levels)
    for L in range(1, levels):
        g = v2d.level_view(pyr, lay, L)[0].cpu().numpy().astype(np.float64)
        assert np.array_equal(g, planes0[L]), L
    # detection: 16x16 grid, k = 256 (the maximum), bit-exact
    border = (win - 1) // 2 + 1
    xy, sc, cnt, _ = v2d.detect_gftt(dev[:1], W, gx, gy, k=k, border=border)
    oxy, osc, ocnt = oracle.detect_gftt(fr[0], gx, gy, k=k, border=border)
    assert np.array_equal(cnt[0].cpu().numpy(), ocnt)
    assert np.array_equal(xy[0].cpu().numpy().reshape(oxy.shape), oxy)
    assert np.array_equal(sc[0].cpu().numpy().reshape(osc.shape), osc)
    # KLT with the largest window through all 8 levels, on a sample of the keypoints
    allp = oxy.reshape(-1, 2)
    allp = allp[allp[:, 0] >= 0]
    rng = np.random.default_rng(5)
    sample = allp[rng.choice(len(allp), 96, replace=False)].astype(np.float32)
    pts = torch.from_numpy(sample[None]).cuda()
    pos, stt, _, _ = v2d.track_klt(dev[:1], pyr[:1], dev[1:], pyr[1:], W, levels, pts, win=win)
    opos, ost, onc, dg = oracle.track_klt(dense0, dense1, W, H, levels, sample, win=win)
    stats = compare_klt(sample, pos[0].cpu().numpy(), stt[0].cpu().numpy(), opos, ost, dg)
    assert stats["pos_over_tol"] == 0 and stats["max_pos_err"] <= POS_TOL, stats
    assert stats["flips_unattributable"] == 0, stats
    assert stats["both_tracked"] >= 48, stats
