"""The KLT parity harness (oracle/parity.py) itself, on hand-made inputs: a
flip is excused only by the margin of the decision that differs, and no
position difference above 0.01 px is excused at all (
SURVEY §8(c) "Tolerances")."""
import numpy as np
import pytest

from oracle import parity as pa

FAR = 1.0  # a margin far outside every band


@pytest.fixture(autouse=True)
def _keep_session():
    """These synthetic failures must not count in the session's parity summary."""
    saved = dict(pa.SESSION)
    yield
    pa.SESSION.clear()
    pa.SESSION.update(saved)


def _diag(ncc=FAR, eig=FAR, bnd=FAR, eps=FAR):
    return np.array([[ncc, eig, bnd, eps]], np.float64)


def _run(gst, ost, diag, gpos=(10.0, 10.0), opos=(10.0, 10.0)):
    return pa.compare_klt(np.array([[5.0, 5.0]], np.float32),
                          np.array([gpos], np.float32), np.array([gst], np.uint8),
                          np.array([opos], np.float64), np.array([ost], np.uint8), diag)


@pytest.mark.parametrize("lost,col", [(pa.LOST_NCC, "ncc"), (pa.LOST_SMALL_EIG, "eig"),
                                      (pa.LOST_OOB, "bnd")])
def test_flip_excused_only_by_its_own_margin(lost, col):
    band = {"ncc": pa.NCC_BAND, "eig": pa.EIG_BAND, "bnd": pa.BOUND_BAND}
    # inside its own band: attributable, both directions
    for g, o in ((pa.TRACKED, lost), (lost, pa.TRACKED)):
        st = _run(g, o, _diag(**{col: 0.5 * band[col]}), gpos=(-1, -1) if g else (10, 10),
                  opos=(-1, -1) if o else (10, 10))
        assert st["flips"] == 1 and st["flips_attributable"] == 1
    # every OTHER margin inside its band, its own far outside: a failure
    others = {k: 0.0 for k in ("ncc", "eig", "bnd", "eps") if k != col}
    with pytest.raises(AssertionError):
        _run(pa.TRACKED, lost, _diag(**{col: FAR}, **others))


def test_lost_lost_flip_uses_either_decision():
    st = _run(pa.LOST_NCC, pa.LOST_OOB, _diag(bnd=1e-4))
    assert st["flips_attributable"] == 1
    st = _run(pa.LOST_NCC, pa.LOST_OOB, _diag(ncc=1e-5))
    assert st["flips_attributable"] == 1
    with pytest.raises(AssertionError):
        _run(pa.LOST_NCC, pa.LOST_OOB, _diag(eig=0.0, eps=0.0))


def test_skipped_never_excused():
    with pytest.raises(AssertionError):
        _run(pa.SKIPPED, pa.TRACKED, _diag(0.0, 0.0, 0.0, 0.0))


def test_position_over_tolerance_never_excused():
    # even with every margin at zero (the old EPS_BAND exemption is gone)
    with pytest.raises(AssertionError):
        _run(pa.TRACKED, pa.TRACKED, _diag(0.0, 0.0, 0.0, 0.0), gpos=(10.011, 10.0))
    st = _run(pa.TRACKED, pa.TRACKED, _diag(), gpos=(10.0, 10.0099))
    assert st["pos_over_tol"] == 0 and st["max_pos_err"] <= pa.POS_TOL


def test_session_counts_accumulate():
    before = dict(pa.SESSION)  # (restored by the fixture afterwards)
    _run(pa.TRACKED, pa.LOST_NCC, _diag(ncc=0.0), opos=(-1, -1))
    assert pa.SESSION["calls"] == before["calls"] + 1
    assert pa.SESSION["flips"] == before["flips"] + 1
    assert pa.SESSION["flips_attributable"] == before["flips_attributable"] + 1
    assert "attributable" in pa.session_summary()
