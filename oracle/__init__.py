"""ORACLE — plain CPU implementation of the cuVSLAM 2D-module hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2506_04359_b200``) never imports it and
shares no code with it.

The arithmetic lives in ``oracle/v2dref.c`` (plain single-threaded C, float64
for KLT, exact integers for pyramid and response; see its header for the
passage each function follows: PAPER.md §2.1 P:53-61 and SURVEY.md §8(c)
D1-D7).  This module is argument marshalling over ctypes only.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "v2dref.c")
_LIB = os.path.join(_HERE, "libv2dref.so")

TRACKED, LOST_OOB, LOST_NCC, LOST_SMALL_EIG, SKIPPED = 0, 1, 2, 3, 4

CFLAGS = ["-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile oracle/v2dref.c into oracle/libv2dref.so (gcc, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", *CFLAGS, "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i, i64, d, f = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_float
        L.v2dref_level_dims.argtypes = [i, i, i, P, P]
        L.v2dref_pyramid_size.argtypes = [i, i, i]
        L.v2dref_pyramid_size.restype = i64
        L.v2dref_build_pyramid.argtypes = [P, i64, i, i, i, P]
        L.v2dref_bilinear.argtypes = [P, i, i, d, d]
        L.v2dref_bilinear.restype = d
        L.v2dref_sobel.argtypes = [P, i, i, P, P]
        L.v2dref_sobel.restype = None
        L.v2dref_lambda_min.argtypes = [d, d, d]
        L.v2dref_lambda_min.restype = d
        L.v2dref_response.argtypes = [P, i64, i, i, P, P]
        L.v2dref_grid_k.argtypes = [i, i, i, i, P]
        L.v2dref_detect_gftt.argtypes = [P, i64, i, i, i, i, i, i, f, i, i, P, P, P, P]
        L.v2dref_ncc.argtypes = [P, P, i]
        L.v2dref_ncc.restype = d
        L.v2dref_track_klt.argtypes = [P, P, i, i, i, P, P, P, i, i, i, d, d, d, i, P, P, P, P]
        L.v2dref_extract_patches.argtypes = [P, i, i, i, P, i, i, P]
        L.v2dref_suppress_mask.argtypes = [P, P, i, d, i, i, P]
        L.v2dref_keyframe_due.argtypes = [i64, i64, d]
        L.v2dref_refill.argtypes = [P, P, i, i, i, P, P, P, P, P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class OracleError(ValueError):
    pass


def _check(rc: int, what: str):
    if rc != 0:
        raise OracleError(f"{what}: invalid argument (rc={rc})")


def level_dims(W: int, H: int, levels: int):
    Ws = np.zeros(8, np.int32)
    Hs = np.zeros(8, np.int32)
    _check(lib().v2dref_level_dims(W, H, levels, _ptr(Ws), _ptr(Hs)), "level_dims")
    return [(int(Ws[L]), int(Hs[L])) for L in range(levels)]


def build_pyramid(img: np.ndarray, levels: int):
    """D1. img: uint8 [H, W] (any row pitch).  Returns a list of float64 planes
    (level 0 first) and the dense concatenation used by track_klt."""
    img = np.ascontiguousarray(img, dtype=np.uint8) if img.strides[1] != 1 else img
    H, W = img.shape
    n = lib().v2dref_pyramid_size(W, H, levels)
    if n < 0:
        raise OracleError("build_pyramid: too many levels for image size")
    out = np.zeros(n, np.float64)
    _check(lib().v2dref_build_pyramid(_ptr(img), img.strides[0], W, H, levels, _ptr(out)),
           "build_pyramid")
    planes, off = [], 0
    for (w, h) in level_dims(W, H, levels):
        planes.append(out[off:off + w * h].reshape(h, w))
        off += w * h
    return planes, out


def sobel(I: np.ndarray):
    """D3 on a float64 plane (clamp-to-edge, Sobel/8)."""
    I = np.ascontiguousarray(I, dtype=np.float64)
    H, W = I.shape
    gx = np.zeros_like(I)
    gy = np.zeros_like(I)
    lib().v2dref_sobel(_ptr(I), W, H, _ptr(gx), _ptr(gy))
    return gx, gy


def bilinear(I: np.ndarray, x: float, y: float) -> float:
    I = np.ascontiguousarray(I, dtype=np.float64)
    H, W = I.shape
    return lib().v2dref_bilinear(_ptr(I), W, H, float(x), float(y))


def lambda_min(a: float, b: float, c: float) -> float:
    return lib().v2dref_lambda_min(float(a), float(b), float(c))


def response(img: np.ndarray, with_exact: bool = False):
    """D4: (R float32 [H,W], lmin float64 [H,W] or None)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape
    R = np.zeros((H, W), np.float32)
    lm = np.zeros((H, W), np.float64) if with_exact else None
    _check(lib().v2dref_response(_ptr(img), img.strides[0], W, H, _ptr(R), _ptr(lm)), "response")
    return R, lm


def grid_k(grid_x: int, grid_y: int, k: int, K_min: int) -> int:
    out = ctypes.c_int(0)
    _check(lib().v2dref_grid_k(grid_x, grid_y, k, K_min, ctypes.byref(out)), "grid_k")
    return out.value


def detect_gftt(img: np.ndarray, grid_x: int, grid_y: int, k: int = 0, K_min: int = 0,
                min_score: float = 0.0, border: int = 3, nms: int = 1,
                mask: np.ndarray | None = None):
    """D5-D6: (kp_xy float32 [gy,gx,k,2], kp_score float32 [gy,gx,k], count int32 [gy*gx])."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape
    kk = grid_k(grid_x, grid_y, k, K_min)
    xy = np.zeros((grid_y, grid_x, kk, 2), np.float32)
    sc = np.zeros((grid_y, grid_x, kk), np.float32)
    cnt = np.zeros(grid_y * grid_x, np.int32)
    if mask is not None:
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        assert mask.shape == img.shape
    _check(lib().v2dref_detect_gftt(_ptr(img), img.strides[0], W, H, grid_x, grid_y, k, K_min,
                                    float(min_score), border, nms, _ptr(mask), _ptr(xy), _ptr(sc),
                                    _ptr(cnt)),
           "detect_gftt")
    return xy, sc, cnt


def ncc(P: np.ndarray, Q: np.ndarray) -> float:
    P = np.ascontiguousarray(P, dtype=np.float64).ravel()
    Q = np.ascontiguousarray(Q, dtype=np.float64).ravel()
    assert P.size == Q.size
    return lib().v2dref_ncc(_ptr(P), _ptr(Q), P.size)


def track_klt(prev_dense: np.ndarray, next_dense: np.ndarray, W: int, H: int, levels: int,
              pts: np.ndarray, guess: np.ndarray | None = None,
              in_status: np.ndarray | None = None, win: int = 21, iters: int = 10,
              eps: float = 0.01, ncc_min: float = 0.8, min_eig: float = 0.01,
              ncc_each_step: bool = False):
    """D7.  prev_dense/next_dense: dense float64 pyramids from build_pyramid()[1].
    Returns (pos float64 [P,2], status uint8 [P], ncc float64 [P], diag float64 [P,4])."""
    pts = np.ascontiguousarray(pts, dtype=np.float32).reshape(-1, 2)
    P = pts.shape[0]
    g = None if guess is None else np.ascontiguousarray(guess, np.float32).reshape(-1, 2)
    s_in = None if in_status is None else np.ascontiguousarray(in_status, np.uint8).ravel()
    pos = np.zeros((P, 2), np.float64)
    st = np.zeros(P, np.uint8)
    nc = np.zeros(P, np.float64)
    dg = np.zeros((P, 4), np.float64)
    _check(lib().v2dref_track_klt(_ptr(prev_dense), _ptr(next_dense), W, H, levels, _ptr(pts),
                                  _ptr(g), _ptr(s_in), P, win, iters, float(eps), float(ncc_min),
                                  float(min_eig), int(ncc_each_step), _ptr(pos), _ptr(st),
                                  _ptr(nc), _ptr(dg)),
           "track_klt")
    return pos, st, nc, dg


def extract_patches(dense_pyr: np.ndarray, W: int, H: int, levels: int, pts: np.ndarray,
                    patch: int = 9):
    """Variant f4: float64 [P, levels, patch, patch]."""
    pts = np.ascontiguousarray(pts, dtype=np.float32).reshape(-1, 2)
    out = np.zeros((pts.shape[0], levels, patch, patch), np.float64)
    _check(lib().v2dref_extract_patches(_ptr(dense_pyr), W, H, levels, _ptr(pts), pts.shape[0],
                                        patch, _ptr(out)), "extract_patches")
    return out


# ---- variant f1 ------------------------------------------------------------
def suppress_mask(tracks: np.ndarray, status: np.ndarray, min_sep: float, W: int, H: int):
    """status: KLT status per track (0 = alive)."""
    tracks = np.ascontiguousarray(tracks, np.float32).reshape(-1, 2)
    status = np.ascontiguousarray(status, np.uint8).ravel()
    mask = np.zeros((H, W), np.uint8)
    _check(lib().v2dref_suppress_mask(_ptr(tracks), _ptr(status), tracks.shape[0],
                                      float(min_sep), W, H, _ptr(mask)), "suppress_mask")
    return mask


def keyframe_due(n_kf: int, n_surv: int, T: float) -> bool:
    return bool(lib().v2dref_keyframe_due(int(n_kf), int(n_surv), float(T)))


def refill(kp_xy, cell_count, k, tracks, status, kf_member, track_id, next_id: int):
    """In place on numpy arrays (tracks f32 [P,2], status/kf_member u8 [P],
    track_id i32 [P]); returns the new next_id."""
    kp_xy = np.ascontiguousarray(kp_xy, np.float32)
    cell_count = np.ascontiguousarray(cell_count, np.int32).ravel()
    nid = np.array([next_id], np.int32)
    _check(lib().v2dref_refill(_ptr(kp_xy), _ptr(cell_count), cell_count.size, k,
                               status.size, _ptr(tracks), _ptr(status), _ptr(kf_member),
                               _ptr(track_id), _ptr(nid)), "refill")
    return int(nid[0])
