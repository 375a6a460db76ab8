"""TEST INFRASTRUCTURE (oracle side): element-by-element comparison of
CUDA-path outputs with the oracle run on the same bytes, used by tests/ and
__graft_entry__.smoke().  Tolerances and ambiguity bands: SURVEY §8(c)
"Tolerances", DESIGN.md §2 / reading #17.

KLT bar (BASELINE north_star: "tracked positions must agree within 0.01 px,
and tracked/lost status must be identical"):
  * every slot TRACKED on both sides agrees within POS_TOL = 0.01 px — no
    exemption of any kind;
  * statuses are identical, except a flip that SURVEY §8(c) attributes to
    rounding: "only if the oracle's deciding quantity lies within its band".
    The deciding quantity is the one of the decision that differs, taken from
    the oracle's per-slot margins (oracle.track_klt's `diag`):
        LOST_NCC       <-> diag[0] = min over levels |NCC_L - ncc_min|      <= 1e-4
        LOST_SMALL_EIG <-> diag[1] = min |lambda/n - min_eig| / (lambda_max/n) <= 1e-5
        LOST_OOB       <-> diag[2] = min distance of an iterate or of the final
                                     position to its bound (px)             <= 1e-3
    A flip TRACKED <-> LOST_X is judged by X's margin alone; LOST_X <-> LOST_Y
    by X's or Y's (both decisions differ).  SKIPPED never flips (it is a pure
    function of the input slot).
Every call adds its counts to SESSION, which tests/conftest.py prints at the
end of the run, so a test log carries the total and attributable flips.
"""
from __future__ import annotations

import numpy as np

import oracle

POS_TOL = 0.01          # px, BASELINE north_star
NCC_BAND = 1e-4         # |NCC - ncc_min|
EIG_BAND = 1e-5         # |lambda/n - min_eig| / (lambda_max/n)
BOUND_BAND = 1e-3       # px to a bound

TRACKED, LOST_OOB, LOST_NCC, LOST_SMALL_EIG, SKIPPED = 0, 1, 2, 3, 4
# status -> (diag column of its deciding quantity, band)
DECISION = {LOST_OOB: (2, BOUND_BAND), LOST_NCC: (0, NCC_BAND), LOST_SMALL_EIG: (1, EIG_BAND)}

SESSION = {"calls": 0, "slots": 0, "both_tracked": 0, "flips": 0, "flips_attributable": 0,
           "pos_over_tol": 0, "max_pos_err": 0.0}


def oracle_pyramid_dense(frame_u8: np.ndarray, W: int, levels: int):
    planes, dense = oracle.build_pyramid(np.ascontiguousarray(frame_u8[:, :W]), levels)
    return planes, dense


def gpu_level_planes(pyr_row: np.ndarray, layout, levels: int):
    out = []
    for L in range(1, levels):
        off, pitch, w, h = layout.offset[L], layout.pitch[L], layout.W[L], layout.H[L]
        out.append(pyr_row[off:off + pitch * h].reshape(h, pitch)[:, :w])
    return out


def flip_attributable(gpu_status: int, oracle_status: int, diag_row) -> bool:
    """True iff the flip gpu_status != oracle_status is explained by the
    oracle's margin of a decision that differs (module docstring)."""
    if gpu_status == oracle_status:
        return True
    kinds = {int(gpu_status), int(oracle_status)} - {TRACKED}
    if SKIPPED in kinds or not kinds <= set(DECISION):
        return False
    return any(diag_row[DECISION[k][0]] <= DECISION[k][1] for k in kinds)


def compare_klt(pts, gpu_pos, gpu_st, ora_pos, ora_st, diag, gpu_ncc=None, ora_ncc=None):
    """Returns a dict of counts; raises AssertionError on any position
    difference > POS_TOL between slots tracked on both sides and on any
    status flip that is not attributable (module docstring)."""
    pts = pts.reshape(-1, 2)
    gpu_pos = gpu_pos.reshape(-1, 2).astype(np.float64)
    gpu_st = gpu_st.ravel()
    ora_pos = ora_pos.reshape(-1, 2)
    ora_st = ora_st.ravel()
    diag = diag.reshape(-1, 4)
    both = (gpu_st == TRACKED) & (ora_st == TRACKED)
    err = np.abs(gpu_pos[both] - ora_pos[both]).max(axis=1) if both.any() else np.zeros(0)
    flips = np.nonzero(gpu_st != ora_st)[0]
    attributable, bad = [], []
    for i in flips:
        (attributable if flip_attributable(gpu_st[i], ora_st[i], diag[i]) else bad).append(int(i))
    far = [int(i) for i in np.nonzero(both)[0][err > POS_TOL]] if both.any() else []
    stats = {
        "n": int(len(gpu_st)), "both_tracked": int(both.sum()),
        "max_pos_err": float(err.max()) if err.size else 0.0,
        "flips": int(len(flips)), "flips_attributable": int(len(attributable)),
        "flips_unattributable": int(len(bad)), "pos_over_tol": int(len(far)),
        "status_hist_gpu": np.bincount(gpu_st, minlength=5).tolist(),
        "status_hist_oracle": np.bincount(ora_st, minlength=5).tolist(),
    }
    SESSION["calls"] += 1
    SESSION["slots"] += stats["n"]
    SESSION["both_tracked"] += stats["both_tracked"]
    SESSION["flips"] += stats["flips"]
    SESSION["flips_attributable"] += stats["flips_attributable"]
    SESSION["pos_over_tol"] += stats["pos_over_tol"]
    SESSION["max_pos_err"] = max(SESSION["max_pos_err"], stats["max_pos_err"])
    if bad or far:
        detail = [(int(i), pts[i].tolist(), int(gpu_st[i]), int(ora_st[i]),
                   gpu_pos[i].tolist(), ora_pos[i].tolist(), diag[i].tolist())
                  for i in (bad + far)[:8]]
        raise AssertionError(f"KLT parity failure: {stats}; examples "
                             f"(slot, pt, gpu_st, oracle_st, gpu_pos, oracle_pos, diag) {detail}")
    return stats


def session_summary() -> str:
    s = SESSION
    return (f"KLT parity summary: {s['calls']} comparisons, {s['slots']} slots, "
            f"{s['both_tracked']} tracked on both sides, max |dpos| {s['max_pos_err']:.3g} px, "
            f"pos > {POS_TOL} px: {s['pos_over_tol']}, status flips: {s['flips']} "
            f"(attributable {s['flips_attributable']}, "
            f"unattributable {s['flips'] - s['flips_attributable']})")
