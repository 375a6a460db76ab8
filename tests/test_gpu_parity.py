"""GPU parity: the CUDA path (through the C ABI) vs the oracle on the same
seeded bytes, element by element.  Bars: pyramid, response and
selection bit-exact; KLT positions <= 0.01 px for slots tracked on both sides
and identical status except rounding-attributable flips inside the stated
bands (oracle/parity.py)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle.parity import POS_TOL, compare_klt, gpu_level_planes

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2506_04359_b200 import vslam2d as v2d


def _to_dev(frames_u8: np.ndarray, pitch: int | None = None):
    """[B, H, W] host u8 -> [B, H, pitch] device (pitch % 16 == 0)."""
    B, H, W = frames_u8.shape
    pitch = pitch or synth.round_up(W, 16)
    t = torch.zeros((B, H, pitch), dtype=torch.uint8)
    t[:, :, :W] = torch.from_numpy(frames_u8)
    return t.cuda()


def _stream(W, H, n, seed, motion=(3.0, 2.0)):
    wl = synth.Workload("t", 7, W, H, 1, 3, motion=motion, stereo_disparity=0.0)
    st = synth.make_stream(wl, n, "cpu", rank_salt=seed)
    return st.frames[0][:, :, :W].numpy().copy(), st


# ------------------------------------------------------------------ pyramid
@pytest.mark.parametrize("W,H,levels", [(640, 480, 3), (752, 480, 4), (1241, 376, 4),
                                        (155, 47, 4), (33, 17, 5), (300, 260, 8), (64, 64, 1),
                                        (1, 1, 1), (129, 2, 2)])
def test_pyramid_bit_exact(W, H, levels):
    rng = np.random.default_rng(W * 7 + H)
    fr = rng.integers(0, 256, (3, H, W), dtype=np.uint8)
    d = _to_dev(fr)
    pyr = v2d.build_pyramid(d, W, levels).cpu().numpy()
    lay = v2d.pyramid_layout(W, H, levels)
    for b in range(3):
        planes, _ = oracle.build_pyramid(fr[b], levels)
        got = gpu_level_planes(pyr[b], lay, levels)
        for L in range(1, levels):
            assert np.array_equal(got[L - 1].astype(np.float64), planes[L]), (b, L)


def test_pyramid_unaligned_pitch_rejected():
    d = torch.zeros((1, 10, 40), dtype=torch.uint8, device="cuda")
    with pytest.raises(v2d.V2DError):
        v2d.build_pyramid(d, 33, 2)  # pitch 40 % 16 != 0


# ---------------------------------------------------------- response/select
@pytest.mark.parametrize("dense", [True, False])
@pytest.mark.parametrize("W,H,seed", [(160, 120, 0), (97, 61, 1), (752, 480, 2)])
def test_response_bit_exact(W, H, seed, dense):
    fr, _ = _stream(W, H, 2, seed)
    d = _to_dev(fr)
    _, _, _, resp = v2d.detect_gftt(d, W, 4, 3, k=8, border=3, want_resp=True, dense=dense)
    resp = resp.cpu().numpy()
    for b in range(fr.shape[0]):
        R, _ = oracle.response(fr[b])
        assert np.array_equal(resp[b], R)


SELECT_CASES = [
    # W, H, gx, gy, k, K_min, border, nms, min_score
    (640, 480, 8, 8, 4, 200, 11, 1, 0.0),
    (752, 480, 8, 8, 0, 1000, 11, 1, 0.0),
    (1241, 376, 8, 8, 0, 2000, 11, 1, 0.0),
    (97, 61, 3, 2, 7, 0, 3, 1, 0.0),
    (97, 61, 3, 2, 7, 0, 3, 0, 0.0),
    (200, 150, 2, 2, 256, 0, 5, 1, 0.0),
    (200, 150, 1, 1, 256, 0, 3, 0, 0.0),
    (333, 111, 7, 5, 3, 0, 11, 1, 50.0),
]


@pytest.mark.parametrize("dense", [True, False])
@pytest.mark.parametrize("W,H,gx,gy,k,K,border,nms,ms", SELECT_CASES)
def test_selection_bit_exact(W, H, gx, gy, k, K, border, nms, ms, dense):
    fr, _ = _stream(W, H, 3, W + H)
    d = _to_dev(fr)
    xy, sc, cnt, _ = v2d.detect_gftt(d, W, gx, gy, k=k, K_min=K, border=border, nms=nms,
                                     min_score=ms, dense=dense)
    xy, sc, cnt = xy.cpu().numpy(), sc.cpu().numpy(), cnt.cpu().numpy()
    for b in range(fr.shape[0]):
        oxy, osc, ocnt = oracle.detect_gftt(fr[b], gx, gy, k=k, K_min=K, min_score=ms,
                                            border=border, nms=nms)
        assert np.array_equal(cnt[b], ocnt)
        assert np.array_equal(xy[b], oxy)
        assert np.array_equal(sc[b], osc)


def test_selection_special_images():
    W, H = 128, 96
    const = np.full((H, W), 90, np.uint8)
    tile = np.zeros((8, 8), np.uint8)
    tile[2:6, 2:6] = 200
    ties = np.tile(tile, (H // 8, W // 8))
    corner = np.full((H, W), 40, np.uint8)
    corner[50:, 70:] = 220
    fr = np.stack([const, ties, corner])
    d = _to_dev(fr)
    xy, sc, cnt, _ = v2d.detect_gftt(d, W, 2, 2, k=40, border=3)
    xy2, sc2, cnt2, _ = v2d.detect_gftt(d, W, 2, 2, k=40, border=3, dense=False)
    assert torch.equal(xy, xy2) and torch.equal(sc, sc2) and torch.equal(cnt, cnt2)
    for b in range(3):
        oxy, osc, ocnt = oracle.detect_gftt(fr[b], 2, 2, k=40, border=3)
        assert np.array_equal(xy[b].cpu().numpy(), oxy)
        assert np.array_equal(sc[b].cpu().numpy(), osc)
        assert np.array_equal(cnt[b].cpu().numpy(), ocnt)
    assert cnt[0].sum().item() == 0


def _extreme_images(W, H):
    """Images at the ends of the response contract's operand ranges (DESIGN.md §5 K2:
    det up to 2^47, D up to 2^49, det = 0 with large trace, tiny det/D)."""
    rng = np.random.default_rng(7)
    yy, xx = np.mgrid[0:H, 0:W]
    return np.stack([
        (((xx + yy) & 1) * 255).astype(np.uint8),            # 1-px checkerboard: Sobel = 0
        ((((xx >> 1) + (yy >> 1)) & 1) * 255).astype(np.uint8),
        (rng.integers(0, 2, (H, W)) * 255).astype(np.uint8),  # binary noise: extreme A, B, C
        rng.integers(0, 2, (H, W)).astype(np.uint8),          # values 0/1: tiny det and D
        ((xx * 255) // (W - 1)).astype(np.uint8),             # horizontal ramp: det = 0
        (((xx + 2 * yy) * 3) % 256).astype(np.uint8),         # diagonal saw: rank-deficient
        np.where(xx > yy, 255, 0).astype(np.uint8),           # saturated diagonal edge
    ])


@pytest.mark.parametrize("dense", [True, False])
def test_response_extreme_ranges(dense):
    W, H = 96, 80
    fr = _extreme_images(W, H)
    d = _to_dev(fr)
    _, _, _, resp = v2d.detect_gftt(d, W, 4, 3, k=8, border=3, want_resp=True, dense=dense)
    xy, sc, cnt, _ = v2d.detect_gftt(d, W, 4, 4, k=16, border=3, dense=dense)
    resp, xy, sc, cnt = (t.cpu().numpy() for t in (resp, xy, sc, cnt))
    for b in range(fr.shape[0]):
        R, _ = oracle.response(fr[b])
        assert np.array_equal(resp[b], R), b
        oxy, osc, ocnt = oracle.detect_gftt(fr[b], 4, 4, k=16, border=3)
        assert np.array_equal(cnt[b], ocnt), b
        assert np.array_equal(xy[b], oxy), b
        assert np.array_equal(sc[b], osc), b
    assert resp[2].max() > 3e4  # binary 0/255 noise: tensor sums near their maximum


def test_detect_rejects_bad_k():
    d = torch.zeros((1, 64, 64), dtype=torch.uint8, device="cuda")
    with pytest.raises(v2d.V2DError):
        v2d.detect_gftt(d, 64, 8, 8, k=4, K_min=256, border=3)  # violates Eq. 1


# ---------------------------------------------------------------------- KLT
def _strict(stats):
    """The KLT bar, asserted explicitly in every KLT test (compare_klt also
    raises): no position of a slot tracked on both sides off by more than
    0.01 px, no status flip outside its own decision's band."""
    assert stats["pos_over_tol"] == 0 and stats["max_pos_err"] <= POS_TOL, stats
    assert stats["flips_unattributable"] == 0, stats
    return stats


def _klt_case(fr_prev, fr_next, W, levels, pts, win=21, iters=10, guess=None, in_status=None,
              eps=0.01, each_step=False):
    B = fr_prev.shape[0]
    dp, dn = _to_dev(fr_prev), _to_dev(fr_next)
    pp = v2d.build_pyramid(dp, W, levels)
    pn = v2d.build_pyramid(dn, W, levels)
    tp = torch.from_numpy(pts).cuda()
    tg = None if guess is None else torch.from_numpy(guess).cuda()
    ti = None if in_status is None else torch.from_numpy(in_status).cuda()
    pos, st, nc, it = v2d.track_klt(dp, pp, dn, pn, W, levels, tp, guess=tg, in_status=ti,
                                    win=win, iters=iters, eps=eps,
                                    flags=v2d.KLT_NCC_EACH_STEP if each_step else 0)
    pos, st, nc = pos.cpu().numpy(), st.cpu().numpy(), nc.cpu().numpy()
    H = fr_prev.shape[1]
    stats = []
    for b in range(B):
        _, d0 = oracle.build_pyramid(fr_prev[b], levels)
        _, d1 = oracle.build_pyramid(fr_next[b], levels)
        opos, ost, onc, dg = oracle.track_klt(
            d0, d1, W, H, levels, pts[b], guess=None if guess is None else guess[b],
            in_status=None if in_status is None else in_status[b], win=win, iters=iters, eps=eps,
            ncc_each_step=each_step)
        stats.append(_strict(compare_klt(pts[b], pos[b], st[b], opos, ost, dg)))
    return stats


def test_klt_c1_pair():
    """BASELINE config C1: 640x480, 3 levels, 8x8 grid, k=4, 21x21 window."""
    f0, f1 = synth.shifted_pair(480, 640, (3.2, -1.7), seed=1)
    xy, _, _ = oracle.detect_gftt(f0, 8, 8, k=4, K_min=200, border=11)
    pts = xy.reshape(1, -1, 2)
    stats = _klt_case(f0[None], f1[None], 640, 3, pts)
    assert stats[0]["both_tracked"] > 200
    assert stats[0]["max_pos_err"] <= 0.01


@pytest.mark.parametrize("win,levels", [(21, 4), (11, 3), (29, 2), (3, 1), (7, 5)])
def test_klt_stream_windows(win, levels):
    W, H = 320, 240
    fr, _ = _stream(W, H, 4, 11 + win, motion=(4.0, 3.0))
    prev, nxt = fr[:-1], fr[1:]
    pts = np.stack([oracle.detect_gftt(f, 4, 4, k=16, border=max(3, (win - 1) // 2 + 1))[0].reshape(-1, 2)
                    for f in prev])
    stats = _klt_case(prev, nxt, W, levels, pts, win=win)
    assert sum(s["both_tracked"] for s in stats) > 0.3 * pts.shape[0] * pts.shape[1]


@pytest.mark.parametrize("win", list(range(3, 31, 2)))
def test_klt_every_window_layout(win):
    """Every window size (each has its own run layout: run length, exactly tiled or
    shifted last run, bank-free patch pitch or the pitch-32 fallback) vs the
    oracle, on a stream with motion and keypoints near the borders."""
    W, H = 160, 120
    levels = 3 if win <= 15 else 2
    fr, _ = _stream(W, H, 3, 101 + win, motion=(3.0, -2.0))
    prev, nxt = fr[:-1], fr[1:]
    pts = np.stack([oracle.detect_gftt(f, 4, 4, k=6, border=max(3, (win - 1) // 2 + 1))[0]
                    .reshape(-1, 2) for f in prev])
    stats = _klt_case(prev, nxt, W, levels, pts, win=win)
    assert sum(s["both_tracked"] for s in stats) > 0.2 * pts.shape[0] * pts.shape[1]


def test_klt_edge_cases():
    W, H = 200, 150
    fr, _ = _stream(W, H, 2, 5)
    pts = np.array([[[-1, -1], [100, 70], [12, 12], [187, 137], [3, 75], [199, 149],
                     [60.25, 40.75], [150, 20], [np.nan, 3], [0, 0]]], np.float32)
    ins = np.array([[0, 1, 0, 0, 0, 0, 0, 0, 0, 0]], np.uint8)
    guess = np.tile(np.array([[[2.5, -1.0]]], np.float32), (1, pts.shape[1], 1))
    _klt_case(fr[:1], fr[1:], W, 3, pts, in_status=ins)
    _klt_case(fr[:1], fr[1:], W, 3, pts, guess=guess)
    # identical frames: zero motion exactly
    d = _to_dev(fr[:1])
    p = v2d.build_pyramid(d, W, 3)
    good = torch.tensor([[[100.0, 70.0], [60.0, 41.0]]], device="cuda")
    pos, st, nc, it = v2d.track_klt(d, p, d, p, W, 3, good)
    assert st.tolist() == [[0, 0]]
    assert torch.equal(pos, good)


def test_klt_rank_deficient_window_and_min_eig_contract():
    """Singular G (vertical stripes: Ty = 0, lambda_min = 0): LOST_SMALL_EIG on
    both sides for any positive min_eig (reading #27); min_eig <= 0 is rejected
    by the ABI (and by the oracle, tests/test_oracle_klt.py)."""
    W, H = 160, 120
    cols = (np.arange(W) * 37 % 251).astype(np.uint8)
    f0 = np.ascontiguousarray(np.tile(cols, (H, 1)))[None]
    pts = np.array([[[80, 60], [50.5, 40.25], [30, 90]]], np.float32)
    for me in (0.01, 1e-30):
        dp = _to_dev(f0)
        pp = v2d.build_pyramid(dp, W, 2)
        pos, st, nc, it = v2d.track_klt(dp, pp, dp, pp, W, 2, torch.from_numpy(pts).cuda(),
                                        min_eig=me)
        assert st.tolist() == [[v2d.LOST_SMALL_EIG] * 3]
        _, d0 = oracle.build_pyramid(f0[0], 2)
        opos, ost, onc, dg = oracle.track_klt(d0, d0, W, H, 2, pts[0], min_eig=me)
        assert ost.tolist() == st[0].tolist()
        _strict(compare_klt(pts[0], pos[0].cpu().numpy(), st[0].cpu().numpy(), opos, ost, dg))
    for me in (0.0, -1.0):
        with pytest.raises(v2d.V2DError):
            v2d.track_klt(dp, pp, dp, pp, W, 2, torch.from_numpy(pts).cuda(), min_eig=me)


def test_klt_track_list_records():
    """The a7 track-list records written by the KLT kernel equal (pos, status,
    ncc) of the same launch, bit for bit."""
    W, H = 320, 240
    fr, _ = _stream(W, H, 2, 21)
    dp, dn = _to_dev(fr[:1]), _to_dev(fr[1:])
    pp, pn = v2d.build_pyramid(dp, W, 3), v2d.build_pyramid(dn, W, 3)
    pts = oracle.detect_gftt(fr[0], 4, 4, k=8, border=11)[0].reshape(1, -1, 2)
    tp = torch.from_numpy(pts).cuda()
    rec = torch.full((1, pts.shape[1], 4), 7.0, device="cuda")
    pos, st, nc, it = v2d.track_klt(dp, pp, dn, pn, W, 3, tp, track_list=rec)
    assert torch.equal(rec[..., :2], pos)
    assert torch.equal(rec[..., 2], st.float())
    assert torch.equal(rec[..., 3], nc)
    with pytest.raises(v2d.V2DError):  # not 16-B aligned
        raw = torch.zeros(4 * pts.shape[1] + 1, device="cuda")
        v2d.track_klt(dp, pp, dn, pn, W, 3, tp, track_list=raw[1:].view(1, -1, 4))


def test_klt_noise_rejects():
    W, H = 320, 240
    fr, _ = _stream(W, H, 1, 3)
    noise = synth.noise_frame(H, W, 99)[None]
    pts = oracle.detect_gftt(fr[0], 4, 4, k=8, border=11)[0].reshape(1, -1, 2)
    stats = _klt_case(fr, noise, W, 3, pts)
    valid = (pts[0, :, 0] >= 0).sum()
    assert stats[0]["status_hist_gpu"][0] <= 0.1 * valid


@pytest.mark.parametrize("win", [21, 11])
def test_klt_variant_ncc_each_step(win):
    """Variant f3 (NCC gate after every Gauss-Newton update) vs the oracle."""
    W, H = 320, 240
    fr, _ = _stream(W, H, 3, 77 + win, motion=(4.0, 3.0))
    prev, nxt = fr[:-1], fr[1:]
    pts = np.stack([oracle.detect_gftt(f, 4, 4, k=16, border=(win - 1) // 2 + 1)[0].reshape(-1, 2)
                    for f in prev])
    stats = _klt_case(prev, nxt, W, 4, pts, win=win, each_step=True)
    assert sum(s["both_tracked"] for s in stats) > 0.3 * pts.shape[0] * pts.shape[1]


def test_klt_rejects_unknown_flags():
    d = torch.zeros((1, 64, 64), dtype=torch.uint8, device="cuda")
    p = v2d.build_pyramid(d, 64, 2)
    with pytest.raises(v2d.V2DError):
        v2d.track_klt(d, p, d, p, 64, 2, torch.zeros((1, 1, 2), device="cuda"), flags=2)


# ------------------------------------------------------------ f4 patches
@pytest.mark.parametrize("W,H,levels,patch", [(320, 240, 4, 9), (97, 61, 3, 9), (200, 150, 2, 5)])
def test_patches_parity(W, H, levels, patch):
    fr, _ = _stream(W, H, 2, W + patch)
    d = _to_dev(fr)
    pyr = v2d.build_pyramid(d, W, levels)
    rng = np.random.default_rng(W)
    pts = np.stack([np.concatenate([rng.uniform(0, [W - 1, H - 1], (40, 2)),
                                    [[-1, -1], [0, 0], [W - 1, H - 1], [5.0, 7.0]]])
                    for _ in range(2)]).astype(np.float32)
    out = v2d.extract_patches(d, pyr, W, levels, torch.from_numpy(pts).cuda(), patch).cpu().numpy()
    for b in range(2):
        _, dense = oracle.build_pyramid(fr[b], levels)
        ref = oracle.extract_patches(dense, W, H, levels, pts[b], patch)
        # fp32 sample positions: |error| <= ulp(max(W,H)) in the bilinear weight,
        # times the largest intensity step (255) + fp32 interpolation rounding
        tol = 255 * float(np.spacing(np.float32(max(W, H)))) + 1e-4
        assert np.abs(out[b] - ref).max() <= tol
        ints = np.all(pts[b] == np.round(pts[b]), axis=1)
        assert np.array_equal(out[b][ints, 0], ref[ints, 0].astype(np.float32))  # L0 exact


# ------------------------------------------------------------ f2 stereo
def test_cross_camera_parity():
    """Variant f2: left -> right tracking with a disparity prior, vs the oracle."""
    W, H = 320, 240
    left, right = synth.stereo_pair(H, W, 20.0, seed=5, occluder=(100, 80, 60, 60))
    pts = oracle.detect_gftt(left, 4, 4, k=12, border=11)[0].reshape(1, -1, 2)
    guess = np.tile(np.array([[[-17.5, 0.5]]], np.float32), (1, pts.shape[1], 1))
    stats = _klt_case(left[None], right[None], W, 3, pts, guess=guess)
    assert stats[0]["both_tracked"] > 0.5 * pts.shape[1]
    # the convenience API is the same kernel with the prior broadcast
    dl, dr = _to_dev(left[None]), _to_dev(right[None])
    pl, pr = v2d.build_pyramid(dl, W, 3), v2d.build_pyramid(dr, W, 3)
    tp = torch.from_numpy(pts).cuda()
    a = v2d.cross_camera_track(dl, pl, dr, pr, W, 3, tp, disparity_prior=(-17.5, 0.5))
    b = v2d.track_klt(dl, pl, dr, pr, W, 3, tp, guess=torch.from_numpy(guess).cuda())
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


# ------------------------------------------------------------ f1 keyframes
def test_keyframe_tracker_stepwise_parity():
    """Variant f1, per frame: the KLT part vs the oracle on the GPU's previous
    table (bands), then the rig-wide Eq. 5 decision, suppression, masked
    detection and refill vs the oracle on the GPU's own KLT output (exact)."""
    from paper_2506_04359_b200.frontend import KeyframeTracker
    W, H, C, levels = 320, 240, 2, 3
    wl = synth.Workload("kf", 12, W, H, C, levels, grid_x=4, grid_y=3, k=6, motion=(7.0, 5.0),
                        stereo_disparity=0.0)
    st = synth.make_stream(wl, 7, "cpu")
    frames = st.frames[:, :, :, :W].numpy().copy()         # [C, T, H, W]
    dev = st.frames.cuda()                                  # [C, T, H, pitch]
    cfg = v2d.FrontendConfig(W=W, H=H, levels=levels, grid_x=4, grid_y=3, k=6, border=11)
    T, ms = 0.9, 8.0
    kt = KeyframeTracker(cfg, C, "cuda", wl.pitch, T=T, min_sep=ms)
    ptr = lambda t: v2d.ptrs_of(dev[:, t])
    kt.start(ptr(0))
    n_kf_frames = 0
    for t in range(1, 7):
        tr0, st0, kf0, id0, nid0 = [x.clone().cpu().numpy() for x in kt.table()]
        kt.step(ptr(t), ptr(t - 1))
        tr1, st1, kf1, id1, nid1 = [x.cpu().numpy() for x in kt.table()]
        flag = int(kt.flag.item())
        refilled = (id1 != id0)
        counts_kf, counts_sv = 0, 0
        pre_tracks, pre_status = tr1.copy(), st1.copy()
        for c in range(C):
            pre_status[c][refilled[c]] = 4
            pre_tracks[c][refilled[c]] = -1
            # KLT part vs oracle (oracle fed the GPU's previous table)
            _, dp = oracle.build_pyramid(frames[c, t - 1], levels)
            _, dc = oracle.build_pyramid(frames[c, t], levels)
            opos, ost, onc, dg = oracle.track_klt(dp, dc, W, H, levels, tr0[c], in_status=st0[c])
            keep = ~refilled[c]
            _strict(compare_klt(tr0[c][keep], pre_tracks[c][keep], pre_status[c][keep],
                                opos[keep], ost[keep], dg[keep]))
            counts_kf += int(kf0[c].sum())
            counts_sv += int((kf0[c].astype(bool) & (pre_status[c] == 0)).sum())
        assert flag == int(oracle.keyframe_due(counts_kf, counts_sv, T))
        n_kf_frames += flag
        for c in range(C):
            otr, ost_, okf, oid = pre_tracks[c].copy(), pre_status[c].copy(), kf0[c].copy(), id0[c].copy()
            onid = int(nid0[c])
            if flag:
                mask = oracle.suppress_mask(otr, ost_, ms, W, H)
                gmask = kt.mask[c, :, :W].cpu().numpy()
                assert np.array_equal(gmask, mask)
                xy, sc, cnt = oracle.detect_gftt(frames[c, t], 4, 3, k=6, border=11, mask=mask)
                assert np.array_equal(kt.kp_xy[c].cpu().numpy(), xy)
                onid = oracle.refill(xy.reshape(-1, 2), cnt, 6, otr, ost_, okf, oid, onid)
            assert np.array_equal(st1[c], ost_) and np.array_equal(id1[c], oid)
            assert np.array_equal(kf1[c], okf) and int(nid1[c]) == onid
            assert np.array_equal(tr1[c][refilled[c]], otr[refilled[c]])
    assert n_kf_frames >= 1


@pytest.mark.parametrize("dense", [True, False])
def test_selection_massive_ties(dense):
    """Thousands of exactly equal responses in one cell (periodic pattern):
    exercises the dense select's tie fallback and the fused kernel's folds."""
    tile = np.zeros((8, 8), np.uint8)
    tile[2:6, 2:6] = 200
    img = np.tile(tile, (64, 64))  # 512 x 512
    d = _to_dev(img[None])
    xy, sc, cnt, _ = v2d.detect_gftt(d, 512, 1, 1, k=256, border=3, dense=dense)
    oxy, osc, ocnt = oracle.detect_gftt(img, 1, 1, k=256, border=3)
    assert np.array_equal(cnt[0].cpu().numpy(), ocnt)
    assert np.array_equal(xy[0].cpu().numpy(), oxy)
    assert np.array_equal(sc[0].cpu().numpy(), osc)


@pytest.mark.parametrize("W,H,gx,gy,k", [(320, 240, 4, 3, 6), (161, 123, 3, 2, 9), (752, 480, 8, 8, 16)])
def test_masked_selection_bit_exact(W, H, gx, gy, k):
    """Masked detection (min_separation suppression): a non-zero mask pixel is not
    eligible but NMS still compares against it; dense and fused paths bit-exact with the
    oracle on random disk masks (the half-resolution candidate map's non-candidate word
    must survive every kernel variant)."""
    wl = synth.Workload("mk", 13, W, H, 2, 1, grid_x=gx, grid_y=gy, k=k, stereo_disparity=0.0)
    st = synth.make_stream(wl, 2, "cpu")
    fr = st.frames[:, 0, :, :W].numpy().copy()
    pitch = synth.round_up(W, 16)
    rng = np.random.default_rng(W + H)
    mask = np.zeros((2, H, pitch), np.uint8)
    for b in range(2):
        for _ in range(max(4, W * H // 3000)):
            x, y, r = rng.integers(0, W), rng.integers(0, H), rng.integers(2, 12)
            yy, xx = np.mgrid[0:H, 0:W]
            mask[b, :, :W][(xx - x) ** 2 + (yy - y) ** 2 < r * r] = 1
    dev = _to_dev(fr, pitch)
    mt = torch.from_numpy(mask).cuda()
    for dense in (True, False):
        xy, sc, cnt, _ = v2d.detect_gftt(dev, W, gx, gy, k=k, border=11, mask=mt, dense=dense)
        for b in range(2):
            oxy, osc, ocnt = oracle.detect_gftt(fr[b], gx, gy, k=k, border=11,
                                                mask=np.ascontiguousarray(mask[b, :, :W]))
            assert np.array_equal(cnt[b].cpu().numpy(), ocnt), (dense, b)
            assert np.array_equal(xy[b].cpu().numpy().reshape(oxy.shape), oxy), (dense, b)
            assert np.array_equal(sc[b].cpu().numpy().reshape(osc.shape), osc), (dense, b)
