"""TEST INFRASTRUCTURE (oracle side): element-by-element comparison of
CUDA-path outputs with the oracle run on the same bytes, used by tests/ and
__graft_entry__.smoke().  Tolerances and ambiguity bands: SURVEY §8(c)
"Tolerances", DESIGN.md §3."""
from __future__ import annotations

import numpy as np

import oracle

POS_TOL = 0.01          # px, BASELINE north_star
NCC_BAND = 1e-4         # |NCC - ncc_min|
EIG_BAND = 1e-5         # |lambda/n - min_eig| / (lambda_max/n)
BOUND_BAND = 1e-3       # px to a bound
EPS_BAND = 2e-3         # |‖eta‖ - eps| (convergence decision; moves positions only)


def oracle_pyramid_dense(frame_u8: np.ndarray, W: int, levels: int):
    planes, dense = oracle.build_pyramid(np.ascontiguousarray(frame_u8[:, :W]), levels)
    return planes, dense


def gpu_level_planes(pyr_row: np.ndarray, layout, levels: int):
    out = []
    for L in range(1, levels):
        off, pitch, w, h = layout.offset[L], layout.pitch[L], layout.W[L], layout.H[L]
        out.append(pyr_row[off:off + pitch * h].reshape(h, pitch)[:, :w])
    return out


def compare_klt(pts, gpu_pos, gpu_st, ora_pos, ora_st, diag, gpu_ncc=None, ora_ncc=None):
    """Returns a dict of counts; raises AssertionError on a non-attributable
    disagreement."""
    pts = pts.reshape(-1, 2)
    gpu_pos = gpu_pos.reshape(-1, 2).astype(np.float64)
    gpu_st = gpu_st.ravel()
    ora_pos = ora_pos.reshape(-1, 2)
    ora_st = ora_st.ravel()
    diag = diag.reshape(-1, 4)
    both = (gpu_st == 0) & (ora_st == 0)
    err = np.abs(gpu_pos[both] - ora_pos[both]).max(axis=1) if both.any() else np.zeros(0)
    flips = np.nonzero(gpu_st != ora_st)[0]
    attributable, bad = [], []
    for i in flips:
        near = (diag[i, 0] <= NCC_BAND) or (diag[i, 1] <= EIG_BAND) or (diag[i, 2] <= BOUND_BAND)
        (attributable if near else bad).append(i)
    far = np.nonzero(both)[0][err > POS_TOL] if both.any() else np.zeros(0, int)
    far_bad = [i for i in far if not ((diag[i, 3] <= EPS_BAND) or (diag[i, 1] <= EIG_BAND) or
                                      (diag[i, 2] <= BOUND_BAND) or (diag[i, 0] <= NCC_BAND))]
    stats = {
        "n": int(len(gpu_st)), "both_tracked": int(both.sum()),
        "max_pos_err": float(err.max()) if err.size else 0.0,
        "flips": int(len(flips)), "flips_attributable": int(len(attributable)),
        "pos_over_tol": int(len(far)), "pos_over_tol_unattributable": int(len(far_bad)),
        "status_hist_gpu": np.bincount(gpu_st, minlength=5).tolist(),
        "status_hist_oracle": np.bincount(ora_st, minlength=5).tolist(),
    }
    if bad or far_bad:
        detail = [(int(i), pts[i].tolist(), int(gpu_st[i]), int(ora_st[i]),
                   gpu_pos[i].tolist(), ora_pos[i].tolist(), diag[i].tolist())
                  for i in (bad + far_bad)[:8]]
        raise AssertionError(f"KLT parity failure: {stats}; examples {detail}")
    return stats
