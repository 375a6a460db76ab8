"""Pins for the oracle's pyramidal LK + NCC gate (D7): exact special cases,
exact integer translations, sub-pixel synthetic shifts with known ground
truth, statistics on decorrelated frames, OpenCV's LK as a loose check, and
the NCC invariants."""
import json
import os

import cv2
import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
H, W, M = 240, 320, 48


def _big(seed, **kw):
    tex = synth.make_texture(H + 2 * M + 8, W + 2 * M + 8, seed, **kw)
    return synth.render(tex, np.zeros((1, 2)), H + 2 * M, W + 2 * M)[0].numpy()


def _int_shift(big, sx, sy):
    """frame1(x, y) = frame0(x - sx, y - sy): an exact integer translation."""
    f0 = big[M:M + H, M:M + W]
    f1 = big[M - sy:M - sy + H, M - sx:M - sx + W]
    return np.ascontiguousarray(f0), np.ascontiguousarray(f1)


def _track(f0, f1, levels, pts=None, **kw):
    _, d0 = oracle.build_pyramid(f0, levels)
    _, d1 = oracle.build_pyramid(f1, levels)
    if pts is None:
        xy, _, _ = oracle.detect_gftt(f0, 4, 4, k=8, border=11)
        pts = xy.reshape(-1, 2)
    return pts, oracle.track_klt(d0, d1, f0.shape[1], f0.shape[0], levels, pts, **kw)


def _interior(p, m=50):
    return (p[:, 0] > m) & (p[:, 0] < W - m) & (p[:, 1] > m) & (p[:, 1] < H - m)


def test_identical_frames_zero_motion_spec():
    f0 = _big(1)[M:M + H, M:M + W].copy()
    pts, (pos, st, nc, dg) = _track(f0, f0, 3)
    valid = pts[:, 0] >= 0
    assert np.all(st[valid] == oracle.TRACKED)
    assert np.array_equal(pos[valid], pts[valid].astype(np.float64))  # exactly
    assert np.all(nc[valid] == pytest.approx(1.0, abs=1e-12))


@pytest.mark.parametrize("sx,sy", [(2, -3), (7, 5), (-13, 9)])
def test_integer_shift_exact(sx, sy):
    """Exact translation at L0: the LK fixed point is the true shift; with a
    tight eps it is reached within 1e-3 px."""
    f0, f1 = _int_shift(_big(5), sx, sy)
    pts, (pos, st, nc, dg) = _track(f0, f1, 3, eps=1e-4)
    ok = (st == oracle.TRACKED) & _interior(pts)
    assert ok.sum() >= 0.6 * _interior(pts).sum()
    err = np.abs(pos[ok] - pts[ok] - [sx, sy])
    assert err.max() < 1e-3
    # with the default eps (0.01 px) the error stays well inside 0.01 px
    pts, (pos, st, nc, dg) = _track(f0, f1, 3)
    ok = (st == oracle.TRACKED)
    assert np.abs(pos[ok] - pts[ok] - [sx, sy]).max() < 5e-3


def test_subpixel_shift_spec():
    """Smooth texture translated by (3.2, -1.7): surviving tracks within 0.1 px
    of ground truth (acceptance criterion 6)."""
    g = GOLD["subpixel_shift"]
    f0, f1 = synth.shifted_pair(H, W, tuple(g["shift"]), seed=7, smooth=True)
    pts, (pos, st, nc, dg) = _track(f0, f1, 3)
    ok = st == oracle.TRACKED
    assert ok.sum() >= 0.9 * (pts[:, 0] >= 0).sum()
    assert np.abs(pos[ok] - pts[ok] - g["shift"]).max() < g["tolerance_px"]


def test_subpixel_shift_textured_c1_shape():
    """Same on the full C1-shaped texture (rectangles included)."""
    f0, f1 = synth.shifted_pair(480, 640, (3.2, -1.7), seed=1)
    xy, _, _ = oracle.detect_gftt(f0, 8, 8, k=4, K_min=200, border=11)
    pts = xy.reshape(-1, 2)
    _, (pos, st, nc, dg) = _track(f0, f1, 3, pts=pts)
    ok = st == oracle.TRACKED
    assert ok.mean() > 0.9
    assert np.abs(pos[ok] - pts[ok] - [3.2, -1.7]).max() < 0.1


def test_convergence_range_spec():
    """Shifts up to ~2^(levels-1) * half_window are recovered on a
    texture smooth at the window scale (sigma 12 px)."""
    big = _big(5, smooth=True, octaves=((12.0, 1.0),))
    for (sx, sy) in [(32, 16), (-28, 20), (0, -34)]:
        f0, f1 = _int_shift(big, sx, sy)
        pts, (pos, st, nc, dg) = _track(f0, f1, 3)
        inner = _interior(pts)
        ok = (st == oracle.TRACKED) & inner
        assert ok.sum() >= 0.8 * inner.sum(), (sx, sy, np.bincount(st[inner]))
        assert np.abs(pos[ok] - pts[ok] - [sx, sy]).max() < 0.1


def test_noise_frame_rejected_spec():
    """Second frame replaced by independent noise: >= 90% lost."""
    f0 = _big(3)[M:M + H, M:M + W].copy()
    f1 = synth.noise_frame(H, W, seed=99)
    pts, (pos, st, nc, dg) = _track(f0, f1, 3)
    valid = pts[:, 0] >= 0
    lost = (st[valid] != oracle.TRACKED).mean()
    assert lost >= GOLD["noise_rejection"]["min_lost_fraction"]
    assert (st[valid] == oracle.LOST_NCC).mean() >= 0.8


def test_agrees_loosely_with_cv2_lk():
    """OpenCV's pyramidal LK (Gaussian pyramid, Scharr) is a loose check only:
    both land within 0.15 px of the truth on a smooth translation."""
    shift = (2.6, 1.3)
    f0, f1 = synth.shifted_pair(H, W, shift, seed=21, smooth=True)
    pts, (pos, st, nc, dg) = _track(f0, f1, 3)
    ok = (st == oracle.TRACKED) & _interior(pts)
    p_cv, st_cv, _ = cv2.calcOpticalFlowPyrLK(f0, f1, pts[ok].reshape(-1, 1, 2), None,
                                             winSize=(21, 21), maxLevel=2)
    good = st_cv.ravel() == 1
    assert good.mean() > 0.9
    ours = pos[ok][good]
    theirs = p_cv.reshape(-1, 2)[good]
    assert np.abs(ours - theirs).max() < 0.15
    assert np.abs(ours - pts[ok][good] - shift).max() < 0.1


def test_ncc_invariants_spec():
    rng = np.random.default_rng(0)
    P = rng.uniform(0, 255, 441)
    assert oracle.ncc(P, P) == pytest.approx(1.0, abs=1e-12)
    assert oracle.ncc(P, -P) == pytest.approx(-1.0, abs=1e-12)
    assert oracle.ncc(P, 3.0 * P + 17.0) == pytest.approx(1.0, abs=1e-12)  # affine invariant
    assert oracle.ncc(np.full(441, 5.0), P) == 0.0  # degenerate denominator
    Q = rng.uniform(0, 255, 441)
    ref = np.corrcoef(P, Q)[0, 1]  # library pin
    assert oracle.ncc(P, Q) == pytest.approx(ref, abs=1e-12)


def test_skipped_and_sentinels():
    f0 = _big(1)[M:M + H, M:M + W].copy()
    pts = np.array([[-1, -1], [100, 100], [120, 80], [np.nan, 5]], np.float32)
    ins = np.array([0, 1, 0, 0], np.uint8)
    _, (pos, st, nc, dg) = _track(f0, f0, 3, pts=pts, in_status=ins)
    assert list(st) == [oracle.SKIPPED, oracle.SKIPPED, oracle.TRACKED, oracle.SKIPPED]
    assert np.all(pos[[0, 1, 3]] == -1.0)


def test_flat_region_small_eig():
    f0 = np.full((H, W), 90, np.uint8)
    f0[:, :40] = np.random.default_rng(0).integers(0, 255, (H, 40), dtype=np.uint8)
    pts = np.array([[200, 120], [20, 120]], np.float32)
    _, (pos, st, nc, dg) = _track(f0, f0, 3, pts=pts)
    assert st[0] == oracle.LOST_SMALL_EIG and st[1] == oracle.TRACKED


def test_rank_deficient_window_small_eig():
    """Vertical stripes: Ty = 0 everywhere, so G = [[a, 0], [0, 0]] is singular
    (lambda_min = 0 exactly).  With any positive min_eig (even 1e-30) the window
    is LOST_SMALL_EIG at L0 and no closed-form solve divides by det = 0."""
    cols = (np.arange(W) * 37 % 251).astype(np.uint8)
    f0 = np.ascontiguousarray(np.tile(cols, (H, 1)))
    pts = np.array([[160, 120], [100.5, 80.25]], np.float32)
    for me in (0.01, 1e-30):
        _, (pos, st, nc, dg) = _track(f0, f0, 2, pts=pts, min_eig=me)
        assert list(st) == [oracle.LOST_SMALL_EIG] * 2
        assert np.all(pos == -1)


@pytest.mark.parametrize("me", [0.0, -0.5, float("nan")])
def test_non_positive_min_eig_rejected(me):
    """Reading #27: min_eig must be > 0 (it is what guarantees det(G) > 0)."""
    f0 = np.full((H, W), 90, np.uint8)
    with pytest.raises(Exception):
        _track(f0, f0, 2, pts=np.array([[100, 100]], np.float32), min_eig=me)


def test_leaving_image_is_oob():
    """A point whose true motion leaves the half-window margin is LOST_OOB."""
    f0, f1 = _int_shift(_big(5), 6, 0)
    pts = np.array([[W - 1 - 10 - 3, 120.0], [150.0, 120.0]], np.float32)
    _, (pos, st, nc, dg) = _track(f0, f1, 3, pts=pts)
    assert st[0] == oracle.LOST_OOB and st[1] == oracle.TRACKED


def test_guess_prior_extends_range():
    big = _big(5)
    f0, f1 = _int_shift(big, 36, 0)
    pts, (pos, st, nc, dg) = _track(f0, f1, 2)
    inner = _interior(pts)
    base = (st[inner] == oracle.TRACKED).mean()
    guess = np.tile(np.array([[35.0, 0.5]], np.float32), (pts.shape[0], 1))
    _, (pos2, st2, nc2, dg2) = _track(f0, f1, 2, pts=pts, guess=guess)
    ok = (st2 == oracle.TRACKED) & inner
    assert ok.mean() / inner.mean() > max(0.9, base)
    assert np.abs(pos2[ok] - pts[ok] - [36, 0]).max() < 0.01


def test_ncc_each_step_variant_is_stricter():
    """Variant f3 (NCC at every optimization step, literal P:61): it adds checks,
    so its TRACKED set is a subset of the per-level reading's, with identical
    positions where both track; on identical frames both agree exactly."""
    for (f0, f1) in [synth.shifted_pair(H, W, (3.2, -1.7), seed=13),
                     (_big(3)[M:M + H, M:M + W].copy(), synth.noise_frame(H, W, 5))]:
        pts, (p0, s0, n0, d0) = _track(f0, f1, 3)
        _, (p1, s1, n1, d1) = _track(f0, f1, 3, pts=pts, ncc_each_step=True)
        t1 = s1 == oracle.TRACKED
        assert np.all(s0[t1] == oracle.TRACKED)
        assert np.array_equal(p1[t1], p0[t1])
    f0 = _big(1)[M:M + H, M:M + W].copy()
    pts, (p0, s0, _, _) = _track(f0, f0, 3)
    _, (p1, s1, _, _) = _track(f0, f0, 3, pts=pts, ncc_each_step=True)
    assert np.array_equal(s0, s1) and np.array_equal(p0, p1)
