"""Pins for variant f2 (cross-camera tracking = the same LK + NCC with a
disparity prior; SPEC S:173-181 worked examples) in the oracle."""
import numpy as np

import oracle
import synth

H, W = 240, 320


def _cross(left, right, levels, guess, pts=None):
    _, dl = oracle.build_pyramid(left, levels)
    _, dr = oracle.build_pyramid(right, levels)
    if pts is None:
        pts = oracle.detect_gftt(left, 4, 4, k=8, border=11)[0].reshape(-1, 2)
    g = np.tile(np.asarray(guess, np.float32), (pts.shape[0], 1))
    return pts, oracle.track_klt(dl, dr, W, H, levels, pts, guess=g)


def test_identical_cameras_match_source_spec():
    """identical cameras at identical pose -> matches equal source positions."""
    left, _ = synth.stereo_pair(H, W, 0.0, seed=1)
    pts, (pos, st, nc, dg) = _cross(left, left, 3, (0.0, 0.0))
    ok = st == oracle.TRACKED
    assert ok.mean() > 0.9 and np.array_equal(pos[ok], pts[ok].astype(np.float64))


def test_disparity_20px_recovered_spec():
    """baseline 0.1 m, depth 2 m, fx 400 -> disparity 20 px recovered within
    0.2 px, seeded with a coarse prior (here 16 px)."""
    d = 400 * 0.1 / 2.0
    left, right = synth.stereo_pair(H, W, d, seed=2, smooth=True)
    pts, (pos, st, nc, dg) = _cross(left, right, 3, (-16.0, 0.0))
    inner = pts[:, 0] > 40
    ok = (st == oracle.TRACKED) & inner
    assert ok.sum() > 0.8 * inner.sum()
    assert np.abs(pos[ok, 0] - pts[ok, 0] + d).max() < 0.2
    assert np.abs(pos[ok, 1] - pts[ok, 1]).max() < 0.2


def test_occluded_feature_lost_spec():
    """a feature occluded in the destination image is lost."""
    left, right = synth.stereo_pair(H, W, 20.0, seed=3, occluder=(100, 80, 80, 80))
    pts = np.array([[160.0, 120.0], [260.0, 60.0]], np.float32)  # inside / outside the block
    _, (pos, st, nc, dg) = _cross(left, right, 3, (-20.0, 0.0), pts=pts)
    assert st[0] != oracle.TRACKED
