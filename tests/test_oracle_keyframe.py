"""Pins for variant f1 (keyframe-driven tracking) in the oracle: SPEC worked
examples of keyframe_due, closed-form suppression disks, an explicit
refill example, masked detection against brute force, and the track-table
invariants of a short keyframe-driven run (lost is terminal, ids unique)."""
import numpy as np
import pytest

import oracle
import synth


@pytest.mark.parametrize("n_kf,n_surv,T,due", [(100, 50, 0.7, True),
                                               (100, 70, 0.7, False),   # S:189 (strict)
                                               (100, 100, 0.99, False),  # S:190 s_curr = s_kf
                                               (0, 0, 0.7, True),       # bootstrap
                                               (3, 2, 0.7, True)])
def test_keyframe_due_spec(n_kf, n_surv, T, due):
    assert oracle.keyframe_due(n_kf, n_surv, T) is due


def test_keyframe_due_monotone():
    """Shrinking the overlap never flips true -> false."""
    for T in (0.3, 0.7, 0.9):
        prev = None
        for ov in range(100, -1, -1):
            d = oracle.keyframe_due(100, ov, T)
            if prev:
                assert d
            prev = d


def test_suppress_mask_closed_form():
    W, H, r = 60, 40, 6.5
    tracks = np.array([[10.25, 12.5], [50.0, 30.0], [30.0, 20.0], [-1, -1]], np.float32)
    status = np.array([0, 0, 2, 4], np.uint8)  # third is lost, fourth empty
    m = oracle.suppress_mask(tracks, status, r, W, H)
    yy, xx = np.mgrid[0:H, 0:W]
    want = np.zeros((H, W), bool)
    for (tx, ty), s in zip(tracks.astype(np.float64), status):
        if s == 0:
            want |= (xx - tx) ** 2 + (yy - ty) ** 2 < r * r
    assert np.array_equal(m.astype(bool), want)


def test_refill_explicit_example():
    k = 2
    kp = np.full((3, k, 2), -1, np.float32)
    kp[0, 0] = [5, 6]
    kp[0, 1] = [7, 8]
    kp[2, 0] = [9, 10]
    cnt = np.array([2, 0, 1], np.int32)
    tracks = np.zeros((6, 2), np.float32)
    status = np.array([0, 4, 2, 0, 1, 4], np.uint8)
    kf = np.zeros(6, np.uint8)
    ids = np.array([3, -1, 1, 2, 0, -1], np.int32)
    nid = oracle.refill(kp.reshape(-1, 2), cnt, k, tracks, status, kf, ids, 4)
    assert nid == 7
    assert tracks[1].tolist() == [5, 6] and tracks[2].tolist() == [7, 8] and tracks[4].tolist() == [9, 10]
    assert status.tolist() == [0, 0, 0, 0, 0, 4]
    assert ids.tolist() == [3, 4, 5, 2, 6, -1]
    assert kf.tolist() == [1, 1, 1, 1, 1, 0]


def test_masked_detection_brute_force():
    img = synth.shifted_pair(96, 128, (0, 0), seed=8)[0]
    xy, sc, cnt = oracle.detect_gftt(img, 2, 2, k=6, border=3)
    zero = np.zeros_like(img)
    xy0, sc0, cnt0 = oracle.detect_gftt(img, 2, 2, k=6, border=3, mask=zero)
    assert np.array_equal(xy, xy0) and np.array_equal(sc, sc0)
    # mask each cell's best keypoint: it disappears and the rest shift up by one
    mask = np.zeros_like(img)
    for cy in range(2):
        for cx in range(2):
            x, y = xy[cy, cx, 0].astype(int)
            mask[y, x] = 1
    xy1, sc1, cnt1 = oracle.detect_gftt(img, 2, 2, k=6, border=3, mask=mask)
    for cy in range(2):
        for cx in range(2):
            n = cnt[cy * 2 + cx]
            assert np.array_equal(xy1[cy, cx, :n - 1], xy[cy, cx, 1:n])
            assert all(mask[int(y), int(x)] == 0 for x, y in xy1[cy, cx, :cnt1[cy * 2 + cx]])


def oracle_keyframe_run(frames, levels, gx, gy, k, T, min_sep, win=21):
    """Reference f1 loop, one camera (tests only): returns per-frame tables."""
    H, W = frames[0].shape
    P = gx * gy * k
    tracks = np.full((P, 2), -1, np.float32)
    status = np.full(P, 4, np.uint8)
    kf = np.zeros(P, np.uint8)
    ids = np.full(P, -1, np.int32)
    nid = 0
    border = (win - 1) // 2 + 1
    xy, sc, cnt = oracle.detect_gftt(frames[0], gx, gy, k=k, border=border)
    nid = oracle.refill(xy.reshape(-1, 2), cnt, k, tracks, status, kf, ids, nid)
    out = [(tracks.copy(), status.copy(), ids.copy(), True)]
    _, prev = oracle.build_pyramid(frames[0], levels)
    for f in frames[1:]:
        _, cur = oracle.build_pyramid(f, levels)
        pos, st, _, _ = oracle.track_klt(prev, cur, W, H, levels, tracks, in_status=status,
                                         win=win)
        tracks = np.where((st == 0)[:, None], pos, -1).astype(np.float32)
        status = st.copy()
        n_kf = int(kf.sum())
        n_surv = int((kf.astype(bool) & (status == 0)).sum())
        due = oracle.keyframe_due(n_kf, n_surv, T)
        if due:
            mask = oracle.suppress_mask(tracks, status, min_sep, W, H)
            xy, sc, cnt = oracle.detect_gftt(f, gx, gy, k=k, border=border, mask=mask)
            nid = oracle.refill(xy.reshape(-1, 2), cnt, k, tracks, status, kf, ids, nid)
        out.append((tracks.copy(), status.copy(), ids.copy(), due))
        prev = cur
    return out


def test_keyframe_run_invariants():
    wl = synth.Workload("kf", 11, 240, 160, 1, 3, motion=(6.0, 4.0), stereo_disparity=0.0)
    st = synth.make_stream(wl, 8, "cpu")
    frames = [st.frames[0, t, :, :wl.W].numpy().copy() for t in range(8)]
    run = oracle_keyframe_run(frames, 3, 3, 2, 4, T=0.9, min_sep=8.0)
    seen = set()
    for t, (tracks, status, ids, due) in enumerate(run):
        alive = status == 0
        assert len(set(ids[alive].tolist())) == alive.sum()  # unique ids
        if t > 0:
            ptr, pst, pids, _ = run[t - 1]
            # a slot keeps its id while alive; an id never reappears after loss
            same = (pst == 0) & alive & (ids == pids)
            reborn = alive & (ids != pids)
            assert np.all(pids[reborn] < ids[reborn])
            for i in ids[reborn]:
                assert i not in seen
        seen |= set(ids[alive].tolist())
    assert run[0][3] and any(d for *_, d in run[1:])  # keyframes happen
