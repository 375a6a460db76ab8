"""Seeded randomized parity (GPU vs oracle): random image sizes, level counts,
windows, grids and keypoint sets (including points at and beyond the borders),
so that combinations the hand-picked cases miss are exercised under the same
bars: pyramid and selection bit-exact, KLT within oracle/parity.py's bands."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle.parity import POS_TOL, compare_klt

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2506_04359_b200 import vslam2d as v2d


def _dev(frames):
    B, H, W = frames.shape
    pitch = synth.round_up(W, 16)
    t = torch.zeros((B, H, pitch), dtype=torch.uint8)
    t[:, :, :W] = torch.from_numpy(frames)
    return t.cuda()


# 200 seeded cases by default (cases 100 and 169 are the flat-window NCC regressions:
# a flat S or T must give NCC 0 as in the oracle).  V2D_FUZZ_CASES=1000 runs more;
# DESIGN.md §2 lists the 4 of 1000 that fail (unconverged tracks at the iteration cap).
@pytest.mark.parametrize("case", range(int(os.environ.get("V2D_FUZZ_CASES", "200"))))
def test_fuzz_detect_and_track(case):
    rng = np.random.default_rng(9000 + case)
    win = int(rng.choice([5, 7, 9, 11, 13, 15, 17, 19, 21]))
    r = (win - 1) // 2
    W = int(rng.integers(2 * r + 24, 260))
    H = int(rng.integers(2 * r + 24, 200))
    max_lv = 1
    while max_lv < 5 and (W >> max_lv) >= 1 and (H >> max_lv) >= 1:
        max_lv += 1
    levels = int(rng.integers(1, max_lv + 1))
    motion = (float(rng.uniform(-3, 3)), float(rng.uniform(-3, 3)))
    wl = synth.Workload("fz", 11, W, H, 1, levels, motion=motion, stereo_disparity=0.0)
    st = synth.make_stream(wl, 3, "cpu", rank_salt=case)
    fr = st.frames[0][:, :, :W].numpy().copy()
    prev, nxt = fr[:2], fr[1:3]
    # pyramid: every level bit-exact
    dp = _dev(prev)
    pp = v2d.build_pyramid(dp, W, levels)
    lay = v2d.pyramid_layout(W, H, levels)
    for b in range(2):
        planes, _ = oracle.build_pyramid(prev[b], levels)
        for L in range(1, levels):
            g = v2d.level_view(pp, lay, L)[b].cpu().numpy().astype(np.float64)
            assert np.array_equal(g, planes[L]), (case, b, L)
    # selection: bit-exact (grid and k random, border = r + 1)
    gx, gy = int(rng.integers(1, 7)), int(rng.integers(1, 6))
    k = int(rng.integers(1, 9))
    border = max(3, r + 1)
    xy, sc, cnt, _ = v2d.detect_gftt(dp, W, gx, gy, k=k, border=border)
    for b in range(2):
        oxy, osc, ocnt = oracle.detect_gftt(prev[b], gx, gy, k=k, border=border)
        assert np.array_equal(cnt[b].cpu().numpy(), ocnt), (case, b)
        assert np.array_equal(xy[b].cpu().numpy().reshape(oxy.shape), oxy), (case, b)
        assert np.array_equal(sc[b].cpu().numpy().reshape(osc.shape), osc), (case, b)
    # KLT: detected points plus random points anywhere (some outside / at the border)
    dn = _dev(nxt)
    pn = v2d.build_pyramid(dn, W, levels)
    extra = np.stack([rng.uniform(-2, W + 1, 12), rng.uniform(-2, H + 1, 12)], 1)
    pts = np.stack([np.concatenate([xy[b].cpu().numpy().reshape(-1, 2), extra])
                    for b in range(2)]).astype(np.float32)
    pos, status, _, _ = v2d.track_klt(dp, pp, dn, pn, W, levels, torch.from_numpy(pts).cuda(),
                                      win=win)
    for b in range(2):
        _, d0 = oracle.build_pyramid(prev[b], levels)
        _, d1 = oracle.build_pyramid(nxt[b], levels)
        opos, ost, onc, dg = oracle.track_klt(d0, d1, W, H, levels, pts[b], win=win)
        stats = compare_klt(pts[b], pos[b].cpu().numpy(), status[b].cpu().numpy(), opos, ost, dg)
        assert stats["pos_over_tol"] == 0 and stats["max_pos_err"] <= POS_TOL, stats
        assert stats["flips_unattributable"] == 0, stats
