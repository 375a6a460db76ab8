"""Pins for the oracle's Eq. 1 rule, eligibility, NMS and per-cell top-k
(D5-D6): SPEC worked examples, brute force on tiny grids, an independent
corner detector (cv2) and invariants."""
import json
import os

import cv2
import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_eq1_spec_example():
    g = GOLD["eq1_k"]
    assert oracle.grid_k(g["N"], g["M"], 0, g["K_I"]) == g["k"]


@pytest.mark.parametrize("gx,gy,k,K,ok", [(8, 8, 4, 255, True), (8, 8, 4, 256, False),
                                          (8, 8, 0, 1000, True), (8, 8, 257, 0, False),
                                          (8, 8, 16, 1000, True), (8, 8, 15, 1000, False),
                                          (0, 8, 1, 0, False)])
def test_eq1_rule(gx, gy, k, K, ok):
    """k > floor(K_I/(N*M)); total k*N*M then exceeds K_I."""
    if ok:
        kk = oracle.grid_k(gx, gy, k, K)
        assert kk > K // (gx * gy) and kk * gx * gy > K
    else:
        with pytest.raises(oracle.OracleError):
            oracle.grid_k(gx, gy, k, K)


def _brute_force(img, gx, gy, k, border, min_score, nms):
    """Independent brute force: candidate list per cell by explicit pixel
    loops over the oracle response (pinned separately), ranked by Python's
    sort on (-score, row-major index) — SPEC's tie-break."""
    R, _ = oracle.response(img)
    H, W = img.shape
    out = {}
    for cy in range(gy):
        for cx in range(gx):
            x0, x1 = cx * W // gx, (cx + 1) * W // gx
            y0, y1 = cy * H // gy, (cy + 1) * H // gy
            c = []
            for y in range(y0, y1):
                for x in range(x0, x1):
                    if not (border <= x <= W - 1 - border and border <= y <= H - 1 - border):
                        continue
                    s = float(R[y, x])
                    if not s > min_score:
                        continue
                    if nms:
                        better = True
                        for j in (-1, 0, 1):
                            for i in (-1, 0, 1):
                                if i == 0 and j == 0:
                                    continue
                                q = float(R[y + j, x + i])
                                qi = (y + j) * W + (x + i)
                                # p must beat q: higher score, or equal score and smaller index
                                if not (s > q or (s == q and y * W + x < qi)):
                                    better = False
                        if not better:
                            continue
                    c.append((-s, y * W + x))
            c.sort()
            out[(cy, cx)] = [(idx % W, idx // W, -ns) for ns, idx in c[:k]]
    return out


@pytest.mark.parametrize("seed,W,H,gx,gy,k,nms", [(0, 48, 40, 3, 2, 5, 1), (1, 37, 29, 4, 3, 7, 1),
                                                  (2, 48, 40, 3, 2, 5, 0), (3, 64, 64, 4, 4, 40, 1)])
def test_topk_brute_force(seed, W, H, gx, gy, k, nms):
    img = synth.shifted_pair(H, W, (0.0, 0.0), seed=seed)[0]
    xy, sc, cnt = oracle.detect_gftt(img, gx, gy, k=k, border=3, nms=nms)
    bf = _brute_force(img, gx, gy, k, 3, 0.0, nms)
    for cy in range(gy):
        for cx in range(gx):
            ref = bf[(cy, cx)]
            assert cnt[cy * gx + cx] == len(ref)
            for s in range(k):
                if s < len(ref):
                    assert (xy[cy, cx, s, 0], xy[cy, cx, s, 1], sc[cy, cx, s]) == \
                        (ref[s][0], ref[s][1], np.float32(ref[s][2]))
                else:
                    assert tuple(xy[cy, cx, s]) == (-1.0, -1.0) and sc[cy, cx, s] == 0.0


def test_ties_break_by_row_major_index():
    """A periodic pattern makes many equal responses; the kept order must be
    ascending row-major index among equal scores."""
    tile = np.zeros((8, 8), np.uint8)
    tile[2:6, 2:6] = 200
    img = np.tile(tile, (6, 8))  # 48 x 64, identical squares
    xy, sc, cnt = oracle.detect_gftt(img, 1, 1, k=64, border=3, nms=1)
    n = cnt[0]
    assert n > 8
    s = sc[0, 0, :n]
    idx = xy[0, 0, :n, 1] * 64 + xy[0, 0, :n, 0]
    for i in range(n - 1):
        assert s[i] > s[i + 1] or (s[i] == s[i + 1] and idx[i] < idx[i + 1])
    assert len(np.unique(s)) < n  # ties really occurred


def test_single_corner_is_top_spec():
    """One bright quadrant corner in a cell: the cell's top keypoint is within
    1 px of the corner, found by an independent brute-force scan of
    cv2.cornerMinEigenVal."""
    img = np.full((64, 64), 40, np.uint8)
    img[30:, 25:] = 220  # corner at (25, 30)
    xy, sc, cnt = oracle.detect_gftt(img, 2, 2, k=1, border=3)
    cell = (30 // 32) * 2 + (25 // 32)
    top = xy.reshape(-1, 1, 2)[cell, 0]
    cvr = cv2.cornerMinEigenVal(img, 3, 3)
    cvr[:3] = cvr[-3:] = 0
    cvr[:, :3] = cvr[:, -3:] = 0
    yb, xb = np.unravel_index(np.argmax(cvr), cvr.shape)
    assert abs(top[0] - xb) <= 1 and abs(top[1] - yb) <= 1
    assert abs(top[0] - 25) <= 1 and abs(top[1] - 30) <= 1


def test_invariants_on_textured_frame():
    img = synth.shifted_pair(200, 260, (0, 0), seed=9)[0]
    for nms in (0, 1):
        xy, sc, cnt = oracle.detect_gftt(img, 5, 4, k=6, border=11, nms=nms)
        xy2, sc2, cnt2 = oracle.detect_gftt(img, 5, 4, k=6, border=11, nms=nms)
        assert np.array_equal(xy, xy2) and np.array_equal(sc, sc2)  # deterministic
        assert np.all(cnt <= 6)  # never more than k per cell
        R, _ = oracle.response(img)
        for cy in range(4):
            for cx in range(5):
                c = cnt[cy * 5 + cx]
                s = sc[cy, cx, :c]
                assert np.all(np.diff(s) <= 0)
                for (x, y), v in zip(xy[cy, cx, :c], s):
                    assert R[int(y), int(x)] == v and v > 0
                    assert cx * 260 // 5 <= x < (cx + 1) * 260 // 5
                    assert cy * 200 // 4 <= y < (cy + 1) * 200 // 4
                    assert 11 <= x <= 260 - 12 and 11 <= y <= 200 - 12
                    if nms:
                        nb = R[int(y) - 1:int(y) + 2, int(x) - 1:int(x) + 2]
                        assert (nb <= v).all()


def test_min_score_filters():
    img = synth.shifted_pair(100, 100, (0, 0), seed=11)[0]
    xy, sc, cnt = oracle.detect_gftt(img, 2, 2, k=50, border=3, min_score=500.0)
    assert np.all(sc[sc != 0] > 500.0)
