"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (device ring, pointer tables, B = F*C camera-frames per launch, the
Frontend2D step): sampled outputs are recomputed by the oracle on the same
bytes — pyramid rows, whole grid cells of the selection, and tracks of sampled
keypoints — under the same bars as tests/test_gpu_parity.py."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle.parity import POS_TOL, compare_klt

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2506_04359_b200 import vslam2d as v2d
    from paper_2506_04359_b200.frontend import Frontend2D, RingSchedule


def _setup(name, F=None, ring=None):
    wl = synth.WORKLOADS[name]
    C = wl.cams
    F = F or max(1, 32 // C)
    ring = ring or 2 * F
    cfg = v2d.FrontendConfig(W=wl.W, H=wl.H, levels=wl.levels, grid_x=wl.grid_x,
                             grid_y=wl.grid_y, k=wl.k, K_min=wl.K_min, border=wl.border,
                             win=wl.win, iters=wl.iters, eps=wl.eps, ncc_min=wl.ncc_min,
                             min_eig=wl.min_eig)
    st = synth.make_stream(wl, ring, "cuda")
    fe = Frontend2D(cfg, C, F, "cuda", wl.pitch)
    sched = RingSchedule(st.frames, F)
    fe.prime(sched.before_first, 1)
    slot0 = fe.kp_xy[0].clone()  # keypoints of frame -1 (the carry overwrites slot 0)
    cur, prev, parity = sched.tables(0)
    fe.step(cur, prev, parity)
    torch.cuda.synchronize()
    fe.tracked_pts = torch.cat([slot0[None], fe.kp_xy[1:-1]], 0)  # [F, C, P, 2]
    return wl, st, fe, sched, F


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_fullsize_sampled_parity(name):
    wl, st, fe, sched, F = _setup(name)
    C = wl.cams
    rng = np.random.default_rng(sum(name.encode()))
    frames = st.frames.cpu().numpy()
    B = F * C
    lay = fe.layout
    samples = sorted(set(rng.choice(B, size=min(2, B), replace=False).tolist()) | {B - 1})
    for b in samples:
        f, c = divmod(b, C)
        cur = frames[c, f % frames.shape[1], :, :wl.W]
        prv = frames[c, (f - 1) % frames.shape[1], :, :wl.W]
        # --- pyramid: sampled rows of every level, bit-exact
        planes, dense_cur = oracle.build_pyramid(cur, wl.levels)
        pyr = fe.pyr[0][b].cpu().numpy()
        for L in range(1, wl.levels):
            g = pyr[lay.offset[L]:lay.offset[L] + lay.pitch[L] * lay.H[L]].reshape(
                lay.H[L], lay.pitch[L])[:, :lay.W[L]]
            rows = rng.choice(lay.H[L], size=min(6, lay.H[L]), replace=False)
            assert np.array_equal(g[rows].astype(np.float64), planes[L][rows]), (name, b, L)
        # --- selection: whole sampled cells, bit-exact
        oxy, osc, ocnt = oracle.detect_gftt(cur, wl.grid_x, wl.grid_y, k=wl.k, K_min=wl.K_min,
                                            border=wl.border)
        gxy = fe.kp_xy[1 + f, c].cpu().numpy().reshape(oxy.shape)
        gsc = fe.kp_score[1 + f, c].cpu().numpy().reshape(osc.shape)
        gcnt = fe.cell_count[1 + f, c].cpu().numpy()
        assert np.array_equal(gcnt, ocnt), (name, b)
        assert np.array_equal(gxy, oxy) and np.array_equal(gsc, osc), (name, b)
        # --- KLT: sampled keypoints of the previous frame tracked prv -> cur
        _, dense_prv = oracle.build_pyramid(prv, wl.levels)
        pts_all = fe.tracked_pts[f, c].cpu().numpy().reshape(-1, 2)
        valid = np.nonzero(pts_all[:, 0] >= 0)[0]
        pick = rng.choice(valid, size=min(96, len(valid)), replace=False)
        opos, ost, onc, dg = oracle.track_klt(dense_prv, dense_cur, wl.W, wl.H, wl.levels,
                                              pts_all[pick], win=wl.win, iters=wl.iters,
                                              eps=wl.eps, ncc_min=wl.ncc_min, min_eig=wl.min_eig)
        gpos = fe.pos[b].cpu().numpy()[pick]
        gst = fe.status[b].cpu().numpy()[pick]
        stats = compare_klt(pts_all[pick], gpos, gst, opos, ost, dg)
        assert stats["pos_over_tol"] == 0 and stats["max_pos_err"] <= POS_TOL, stats
        assert stats["flips_unattributable"] == 0, stats
        assert stats["both_tracked"] > 0.5 * len(pick), stats


def test_fullsize_tracking_quality_c2():
    """Property at full size: tracked displacements match the generator's true
    motion (Catmull-Rom rendering, so within ~0.1 px) for most tracks."""
    wl, st, fe, sched, F = _setup("c2")
    C = wl.cams
    pos = fe.pos.cpu().numpy()
    status = fe.status.cpu().numpy()
    pts = fe.tracked_pts.cpu().numpy().reshape(F * C, -1, 2)
    errs = []
    for b in range(F * C):
        f, c = divmod(b, C)
        true = st.true_displacement(c, f)
        ok = status[b] == 0
        errs.append(np.abs(pos[b][ok] - pts[b][ok] - true).max(axis=1))
    e = np.concatenate(errs)
    assert len(e) > 0.8 * F * C * fe.P * 0.5
    assert np.median(e) < 0.05 and np.mean(e < 0.2) > 0.95


@pytest.mark.parametrize("name,F,steps", [("c2", 4, 4), ("c5", 1, 3)])
def test_multistep_stream_parity(name, F, steps):
    """Several consecutive steps of the bench configuration (pyramid parity double
    buffer, keypoint carry from the last frame of a step to the first of the
    next): sampled selections and tracks of every step agree with the oracle."""
    wl = synth.WORKLOADS[name]
    C = wl.cams
    cfg = v2d.FrontendConfig(W=wl.W, H=wl.H, levels=wl.levels, grid_x=wl.grid_x,
                             grid_y=wl.grid_y, k=wl.k, K_min=wl.K_min, border=wl.border,
                             win=wl.win, iters=wl.iters, eps=wl.eps, ncc_min=wl.ncc_min,
                             min_eig=wl.min_eig)
    st = synth.make_stream(wl, 2 * F * steps, "cuda")
    fe = Frontend2D(cfg, C, F, "cuda", wl.pitch)
    sched = RingSchedule(st.frames, F)
    frames = st.frames.cpu().numpy()
    R = frames.shape[1]
    rng = np.random.default_rng(7)
    fe.prime(sched.before_first, 1)
    for s in range(steps):
        slot0 = fe.kp_xy[0].clone()  # carry from step s-1 (overwritten by this step's carry)
        cur, prev, parity = sched.tables(s)
        fe.step(cur, prev, parity)
        torch.cuda.synchronize()
        pts_in = torch.cat([slot0[None], fe.kp_xy[1:-1]], 0)  # frame f tracks slot f
        b = int(rng.integers(F * C))
        f, c = divmod(b, C)
        t = s * F + f
        img, prv = frames[c, t % R, :, :wl.W], frames[c, (t - 1) % R, :, :wl.W]
        oxy, osc, ocnt = oracle.detect_gftt(img, wl.grid_x, wl.grid_y, k=wl.k, K_min=wl.K_min,
                                            border=wl.border)
        assert np.array_equal(fe.kp_xy[1 + f, c].cpu().numpy().reshape(oxy.shape), oxy), (s, b)
        assert np.array_equal(fe.cell_count[1 + f, c].cpu().numpy(), ocnt), (s, b)
        _, d0 = oracle.build_pyramid(prv, wl.levels)
        _, d1 = oracle.build_pyramid(img, wl.levels)
        pts = pts_in[f, c].cpu().numpy().reshape(-1, 2)
        valid = np.nonzero(pts[:, 0] >= 0)[0]
        pick = rng.choice(valid, size=min(64, len(valid)), replace=False)
        opos, ost, onc, dg = oracle.track_klt(d0, d1, wl.W, wl.H, wl.levels, pts[pick],
                                              win=wl.win, iters=wl.iters, eps=wl.eps,
                                              ncc_min=wl.ncc_min, min_eig=wl.min_eig)
        stats = compare_klt(pts[pick], fe.pos[b].cpu().numpy()[pick],
                            fe.status[b].cpu().numpy()[pick], opos, ost, dg)
        assert stats["pos_over_tol"] == 0 and stats["max_pos_err"] <= POS_TOL, stats
        assert stats["flips_unattributable"] == 0, stats
        assert stats["both_tracked"] > 0.5 * len(pick), (s, stats)


@pytest.mark.parametrize("name,win,each", [("c5", 11, False), ("c5", 13, False),
                                           ("c4", 11, True), ("c5", 21, True)])
def test_fullsize_klt_variants_sampled(name, win, each):
    """The f3 variants at full size on the bench data: the two-keypoints-per-warp
    kernel (windows <= 13) and NCC at every Gauss-Newton step, sampled keypoints
    of sampled images recomputed by the oracle, strict KLT bar."""
    wl, st, fe, sched, F = _setup(name)
    C = wl.cams
    B = F * C
    frames = st.frames.cpu().numpy()
    cur, prev, parity = sched.tables(0)
    pts = fe.tracked_pts.reshape(B, fe.P, 2).contiguous()
    pos, stt, nc, it = (torch.empty_like(fe.pos), torch.empty_like(fe.status),
                        torch.empty_like(fe.ncc), torch.empty_like(fe.iters))
    v2d.track_klt_ptrs(prev, fe.prev_pyr_ptrs[parity], cur, fe.pyr_ptrs[parity], fe.pitch, B,
                       wl.W, wl.H, wl.levels, pts, None, None, fe.P, win, wl.iters, wl.eps,
                       wl.ncc_min, wl.min_eig, pos, stt, nc, it,
                       v2d.KLT_NCC_EACH_STEP if each else 0)
    torch.cuda.synchronize()
    rng = np.random.default_rng(win * 31 + each)
    for b in sorted(set(rng.choice(B, size=2, replace=False).tolist())):
        f, c = divmod(b, C)
        _, d_prv = oracle.build_pyramid(frames[c, (f - 1) % frames.shape[1], :, :wl.W], wl.levels)
        _, d_cur = oracle.build_pyramid(frames[c, f % frames.shape[1], :, :wl.W], wl.levels)
        pa = pts[b].cpu().numpy()
        valid = np.nonzero(pa[:, 0] >= 0)[0]
        pick = rng.choice(valid, size=min(80, len(valid)), replace=False)
        opos, ost, onc, dg = oracle.track_klt(d_prv, d_cur, wl.W, wl.H, wl.levels, pa[pick],
                                              win=win, iters=wl.iters, eps=wl.eps,
                                              ncc_min=wl.ncc_min, min_eig=wl.min_eig,
                                              ncc_each_step=each)
        stats = compare_klt(pa[pick], pos[b].cpu().numpy()[pick], stt[b].cpu().numpy()[pick],
                            opos, ost, dg)
        assert stats["pos_over_tol"] == 0 and stats["max_pos_err"] <= POS_TOL, stats
        assert stats["flips_unattributable"] == 0, stats
        assert stats["both_tracked"] > 0.5 * len(pick), stats
