"""Pins for variant f4 (per-level 9x9 patches) in the oracle:
closed forms against direct slicing of the (pinned) pyramid levels."""
import numpy as np

import oracle
import synth


def test_patches_integer_centres_equal_slices():
    img = synth.shifted_pair(96, 128, (0, 0), seed=2)[0]
    planes, dense = oracle.build_pyramid(img, 3)
    # for each level pick the keypoint whose level-L centre c_L = (p+0.5)/2^L - 0.5
    # is an integer: the patch is then a plain slice of the level plane
    for L in range(3):
        s = 1 << L
        cx, cy = 12, 9                      # level-L integer centre
        px, py = (cx + 0.5) * s - 0.5, (cy + 0.5) * s - 0.5
        out = oracle.extract_patches(dense, 128, 96, 3, np.array([[px, py]], np.float32))
        want = planes[L][cy - 4:cy + 5, cx - 4:cx + 5]
        assert np.array_equal(out[0, L], want)


def test_patches_clamp_edge_and_empty():
    img = synth.shifted_pair(40, 50, (0, 0), seed=3)[0]
    planes, dense = oracle.build_pyramid(img, 2)
    out = oracle.extract_patches(dense, 50, 40, 2, np.array([[1, 2], [-1, -1]], np.float32))
    pad = np.pad(planes[0], 4, mode="edge")
    assert np.array_equal(out[0, 0], pad[2 - 4 + 4:2 + 5 + 4, 1 - 4 + 4:1 + 5 + 4])
    assert np.all(out[1] == 0)
    const = np.full((40, 50), 77, np.uint8)
    _, d = oracle.build_pyramid(const, 2)
    o = oracle.extract_patches(d, 50, 40, 2, np.array([[10.3, 20.7]], np.float32))
    assert np.all(o == 77)


def test_patches_subpixel_is_bilinear():
    img = synth.shifted_pair(60, 70, (0, 0), seed=4)[0]
    planes, dense = oracle.build_pyramid(img, 1)
    x, y = 30.25, 20.5
    out = oracle.extract_patches(dense, 70, 60, 1, np.array([[x, y]], np.float32))
    I = planes[0]
    for (v, u) in [(0, 0), (4, 4), (8, 3)]:
        xx, yy = x + u - 4, y + v - 4
        x0, y0 = int(np.floor(xx)), int(np.floor(yy))
        a, b = xx - x0, yy - y0
        want = ((1 - b) * ((1 - a) * I[y0, x0] + a * I[y0, x0 + 1]) +
                b * ((1 - a) * I[y0 + 1, x0] + a * I[y0 + 1, x0 + 1]))
        assert abs(out[0, 0, v, u] - want) < 1e-12
