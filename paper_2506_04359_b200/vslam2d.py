"""Thin Python binding of the C ABI in include/vslam2d.h (ctypes).

Argument marshalling only: every step of the path runs in the sm_100a kernels
of libvslam2d.so.  There is no CPU fallback — importing this module on a box
without the built library raises, and every call requires CUDA tensors.

Function names mirror the C ABI (v2d_build_pyramid -> build_pyramid, ...).
All calls are enqueued on torch.cuda.current_stream() and return without
synchronising.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

from . import build as _build

LIB_PATH = _build.LIB

TRACKED, LOST_OOB, LOST_NCC, LOST_SMALL_EIG, SKIPPED = 0, 1, 2, 3, 4
KLT_NCC_EACH_STEP = 1
MAX_LEVELS, MAX_K, MAX_WIN = 8, 256, 29


class V2DError(RuntimeError):
    pass


class Layout(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int), ("W", ctypes.c_int * 8), ("H", ctypes.c_int * 8),
                ("pitch", ctypes.c_int64 * 8), ("offset", ctypes.c_int64 * 8),
                ("floats_per_image", ctypes.c_int64)]


_SYMBOLS = ("v2d_pyramid_layout", "v2d_grid_k", "v2d_build_pyramid", "v2d_detect_gftt",
            "v2d_track_klt", "v2d_extract_patches", "v2d_suppress_mask", "v2d_track_survival",
            "v2d_keyframe_decide", "v2d_refill_tracks", "v2d_strerror", "v2d_version",
            "v2d_keyframe_decide_graph", "v2d_ring_tables", "v2d_survival_decide")

_lib = None


def load() -> ctypes.CDLL:
    """Load libvslam2d.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2506_04359_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    vp, i, i64, f = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float
    L.v2d_pyramid_layout.argtypes = [i, i, i, ctypes.POINTER(Layout)]
    L.v2d_grid_k.argtypes = [i, i, i, i, ctypes.POINTER(ctypes.c_int)]
    L.v2d_build_pyramid.argtypes = [vp, i64, i, i, i, i, vp, vp]
    L.v2d_detect_gftt.argtypes = [vp, i64, i, i, i, i, i, i, i, f, i, i, vp, vp, vp, vp, vp, vp,
                                  vp, vp]
    L.v2d_suppress_mask.argtypes = [vp, vp, i, i, f, i, i, vp, i64, vp, vp]
    L.v2d_track_survival.argtypes = [vp, vp, i, i, vp, vp]
    L.v2d_keyframe_decide.argtypes = [vp, i, f, vp, vp, vp]
    L.v2d_keyframe_decide_graph.argtypes = [vp, i, f, vp, vp, vp, ctypes.c_uint64, vp]
    L.v2d_ring_tables.argtypes = [vp, i, i, vp, vp, vp, vp]
    L.v2d_survival_decide.argtypes = [vp, vp, i, i, vp, f, vp, vp, vp, ctypes.c_uint64, vp, vp]
    L.v2d_refill_tracks.argtypes = [vp, vp, i, i, i, vp, i, i, vp, vp, vp, vp, vp, vp]
    L.v2d_track_klt.argtypes = [vp, vp, vp, vp, i64, i, i, i, i, vp, vp, vp, i, i, i, f, f, f,
                                vp, vp, vp, vp, vp, ctypes.c_uint, vp]
    L.v2d_extract_patches.argtypes = [vp, vp, i64, i, i, i, i, vp, i, i, vp, vp]
    L.v2d_strerror.argtypes = [i]
    L.v2d_strerror.restype = ctypes.c_char_p
    L.v2d_version.restype = i
    _lib = L
    return L


def exported_symbols() -> list[str]:
    L = load()
    return [s for s in _SYMBOLS if hasattr(L, s)]


def _check(rc: int, what: str):
    if rc != 0:
        raise V2DError(f"{what}: {load().v2d_strerror(rc).decode()} (rc={rc})")


def _p(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise V2DError("vslam2d: tensors must live on a CUDA device (no CPU fallback)")


# --------------------------------------------------------------------------
# host helpers
# --------------------------------------------------------------------------
def pyramid_layout(W: int, H: int, levels: int) -> Layout:
    out = Layout()
    _check(load().v2d_pyramid_layout(W, H, levels, ctypes.byref(out)), "pyramid_layout")
    return out


def grid_k(grid_x: int, grid_y: int, k: int, K_min: int) -> int:
    out = ctypes.c_int(0)
    _check(load().v2d_grid_k(grid_x, grid_y, k, K_min, ctypes.byref(out)), "grid_k")
    return out.value


def ptr_table(addrs, device) -> torch.Tensor:
    """Device int64 array holding the given byte addresses (host arithmetic, one
    H2D copy: no kernel launches)."""
    host = torch.tensor([int(a) for a in addrs], dtype=torch.int64)
    return host.to(device)


def ptrs_of(t: torch.Tensor) -> torch.Tensor:
    """Device int64 array of per-image base pointers of a batched tensor
    t[B, ...] (addresses computed on the host, one H2D copy, no kernels)."""
    stride = t.stride(0) * t.element_size()
    base = t.data_ptr()
    return ptr_table((base + i * stride for i in range(t.shape[0])), t.device)


def level_view(pyr: torch.Tensor, lay: Layout, L: int) -> torch.Tensor:
    """[B, H_L, W_L] view of level L (>= 1) of batched pyramids pyr[B, floats]."""
    off, pitch, w, h = lay.offset[L], lay.pitch[L], lay.W[L], lay.H[L]
    return pyr[:, off:off + pitch * h].view(pyr.shape[0], h, pitch)[:, :, :w]


# --------------------------------------------------------------------------
# pointer-array entry points (1:1 with the C ABI)
# --------------------------------------------------------------------------
def build_pyramid_ptrs(l0_ptrs, l0_pitch, B, W, H, levels, pyr_ptrs):
    _check(load().v2d_build_pyramid(_p(l0_ptrs), l0_pitch, B, W, H, levels, _p(pyr_ptrs),
                                    _stream()), "build_pyramid")


def workspace_pitch(W: int) -> int:
    """Row pitch (floats) of the dense-detection workspace."""
    return (W + 31) // 32 * 32


def detect_gftt_ptrs(l0_ptrs, l0_pitch, B, W, H, grid_x, grid_y, k, K_min, min_score, border,
                     nms, kp_xy, kp_score, cell_count, resp=None, mask_ptrs=None, enable=None,
                     workspace=None):
    _need_cuda(kp_xy, kp_score, cell_count, resp, enable, workspace)
    if workspace is not None and workspace.numel() < B * H * workspace_pitch(W):
        raise V2DError("detect_gftt: workspace needs B*H*round_up(W,32) floats")
    _check(load().v2d_detect_gftt(_p(l0_ptrs), l0_pitch, B, W, H, grid_x, grid_y, k, K_min,
                                  float(min_score), border, nms, _p(kp_xy), _p(kp_score),
                                  _p(cell_count), _p(resp), _p(workspace), _p(mask_ptrs),
                                  _p(enable), _stream()), "detect_gftt")


def track_klt_ptrs(prev_l0_ptrs, prev_pyr_ptrs, next_l0_ptrs, next_pyr_ptrs, l0_pitch, B, W, H,
                   levels, pts, guess, in_status, P, win, iters, eps, ncc_min, min_eig, out_pos,
                   status, ncc=None, iters_out=None, flags=0, track_list=None):
    _need_cuda(pts, guess, in_status, out_pos, status, ncc, iters_out, track_list)
    _check(load().v2d_track_klt(_p(prev_l0_ptrs), _p(prev_pyr_ptrs), _p(next_l0_ptrs),
                                _p(next_pyr_ptrs), l0_pitch, B, W, H, levels, _p(pts), _p(guess),
                                _p(in_status), P, win, iters, float(eps), float(ncc_min),
                                float(min_eig), _p(out_pos), _p(status), _p(ncc), _p(iters_out),
                                _p(track_list), int(flags), _stream()), "track_klt")


# --------------------------------------------------------------------------
# tensor-level conveniences
# --------------------------------------------------------------------------
def _frames(frames: torch.Tensor):
    """frames: uint8 CUDA [B, H, pitch] (pitch % 16 == 0, contiguous rows)."""
    _need_cuda(frames)
    if frames.dtype != torch.uint8 or frames.dim() != 3 or frames.stride(2) != 1:
        raise V2DError("frames must be uint8 [B, H, pitch] with unit column stride")
    return frames.shape[0], frames.shape[1], frames.stride(1)


def build_pyramid(frames: torch.Tensor, W: int, levels: int, out: torch.Tensor | None = None):
    """Pyramids of B frames -> fp32 [B, floats_per_image] (levels 1..L-1)."""
    B, H, pitch = _frames(frames)
    lay = pyramid_layout(W, H, levels)
    n = max(int(lay.floats_per_image), 32)
    if out is None:
        out = torch.empty((B, n), dtype=torch.float32, device=frames.device)
    build_pyramid_ptrs(ptrs_of(frames), pitch, B, W, H, levels, ptrs_of(out))
    return out


def detect_gftt(frames: torch.Tensor, W: int, grid_x: int, grid_y: int, k: int = 0,
                K_min: int = 0, min_score: float = 0.0, border: int = 11, nms: int = 1,
                want_resp: bool = False, mask: torch.Tensor | None = None,
                dense: bool = True):
    """-> (kp_xy [B,gy,gx,k,2], kp_score [B,gy,gx,k], cell_count [B,gy*gx], resp|None)."""
    B, H, pitch = _frames(frames)
    kk = grid_k(grid_x, grid_y, k, K_min)
    dev = frames.device
    xy = torch.empty((B, grid_y, grid_x, kk, 2), dtype=torch.float32, device=dev)
    sc = torch.empty((B, grid_y, grid_x, kk), dtype=torch.float32, device=dev)
    cnt = torch.empty((B, grid_y * grid_x), dtype=torch.int32, device=dev)
    resp = torch.empty((B, H, W), dtype=torch.float32, device=dev) if want_resp else None
    if mask is not None and (mask.shape != frames.shape or mask.dtype != torch.uint8):
        raise V2DError("mask must be uint8 with the frames' shape [B, H, pitch]")
    ws = torch.empty((B, H, workspace_pitch(W)), dtype=torch.float32, device=dev) if dense else None
    detect_gftt_ptrs(ptrs_of(frames), pitch, B, W, H, grid_x, grid_y, k, K_min, min_score,
                     border, nms, xy, sc, cnt, resp, None if mask is None else ptrs_of(mask),
                     None, ws)
    return xy, sc, cnt, resp


def track_klt(prev_frames, prev_pyr, next_frames, next_pyr, W: int, levels: int,
              pts: torch.Tensor, guess=None, in_status=None, win: int = 21, iters: int = 10,
              eps: float = 0.01, ncc_min: float = 0.8, min_eig: float = 0.01, flags: int = 0,
              track_list: torch.Tensor | None = None):
    """pts [B, P, 2] -> (pos [B,P,2], status u8 [B,P], ncc [B,P], iters int32 [B,P]);
    track_list (optional fp32 [B,P,4]) also receives the (x, y, status, ncc) records."""
    B, H, pitch = _frames(prev_frames)
    _frames(next_frames)
    P = pts.shape[1]
    dev = pts.device
    pts = pts.contiguous().float()
    pos = torch.empty((B, P, 2), dtype=torch.float32, device=dev)
    st = torch.empty((B, P), dtype=torch.uint8, device=dev)
    nc = torch.empty((B, P), dtype=torch.float32, device=dev)
    it = torch.empty((B, P), dtype=torch.int32, device=dev)
    track_klt_ptrs(ptrs_of(prev_frames), ptrs_of(prev_pyr), ptrs_of(next_frames),
                   ptrs_of(next_pyr), pitch, B, W, H, levels, pts,
                   None if guess is None else guess.contiguous().float(),
                   None if in_status is None else in_status.contiguous(), P, win, iters, eps,
                   ncc_min, min_eig, pos, st, nc, it, flags, track_list)
    return pos, st, nc, it


@dataclass
class FrontendConfig:
    W: int
    H: int
    levels: int
    grid_x: int = 8
    grid_y: int = 8
    k: int = 0
    K_min: int = 0
    min_score: float = 0.0
    border: int = 11
    nms: int = 1
    win: int = 21
    iters: int = 10
    eps: float = 0.01
    ncc_min: float = 0.8
    min_eig: float = 0.01
    klt_flags: int = 0


def extract_patches_ptrs(l0_ptrs, pyr_ptrs, l0_pitch, B, W, H, levels, pts, P, patch, out):
    _need_cuda(pts, out)
    _check(load().v2d_extract_patches(_p(l0_ptrs), _p(pyr_ptrs), l0_pitch, B, W, H, levels,
                                      _p(pts), P, patch, _p(out), _stream()), "extract_patches")


def extract_patches(frames, pyr, W: int, levels: int, pts: torch.Tensor, patch: int = 9):
    """Variant f4: [B, P, levels, patch, patch] fp32 patches."""
    B, H, pitch = _frames(frames)
    P = pts.shape[1]
    out = torch.empty((B, P, levels, patch, patch), dtype=torch.float32, device=pts.device)
    extract_patches_ptrs(ptrs_of(frames), ptrs_of(pyr), pitch, B, W, H, levels,
                         pts.contiguous().float(), P, patch, out)
    return out


def cross_camera_track(src_frames, src_pyr, dst_frames, dst_pyr, W: int, levels: int,
                       pts: torch.Tensor, disparity_prior=(0.0, 0.0), **kw):
    """Variant f2 ("cross-camera
    (left-to-right) tracking"): the same pyramidal LK + NCC kernel between two
    synchronized cameras, seeded with a disparity prior (dst = src + prior)."""
    B, P = pts.shape[0], pts.shape[1]
    guess = torch.tensor(disparity_prior, dtype=torch.float32, device=pts.device)
    guess = guess.view(1, 1, 2).expand(B, P, 2).contiguous()
    return track_klt(src_frames, src_pyr, dst_frames, dst_pyr, W, levels, pts, guess=guess, **kw)


# --------------------------------------------------------------------------
# variant f1: keyframe-driven continuous tracking
# --------------------------------------------------------------------------
def suppress_mask_ptrs(tracks, status, B, P, min_sep, W, H, mask_ptrs, mask_pitch, enable=None):
    _need_cuda(tracks, status, enable)
    _check(load().v2d_suppress_mask(_p(tracks), _p(status), B, P, float(min_sep), W, H,
                                    _p(mask_ptrs), mask_pitch, _p(enable), _stream()),
           "suppress_mask")


def track_survival(status, kf_member, counts):
    B, P = status.shape
    _need_cuda(status, kf_member, counts)
    _check(load().v2d_track_survival(_p(status), _p(kf_member), B, P, _p(counts), _stream()),
           "track_survival")


def keyframe_decide(counts, T, flag, totals=None):
    _need_cuda(counts, flag, totals)
    _check(load().v2d_keyframe_decide(_p(counts), counts.shape[0], float(T), _p(flag),
                                      _p(totals), _stream()), "keyframe_decide")


def keyframe_decide_graph(counts, T, flag, totals=None, kf_count=None, cond_handle: int = 0):
    """v2d_keyframe_decide_graph: the decision, the device keyframe counter and (inside a
    captured graph) the conditional node's value."""
    _need_cuda(counts, flag, totals, kf_count)
    _check(load().v2d_keyframe_decide_graph(_p(counts), counts.shape[0], float(T), _p(flag),
                                            _p(totals), _p(kf_count), int(cond_handle),
                                            _stream()), "keyframe_decide_graph")


def survival_decide(status, kf_member, counts, T, flag, done, totals=None, kf_count=None,
                    cond_handle: int = 0):
    """v2d_survival_decide: per-image survival counts and the rig-wide Eq. 5 decision in
    one launch (done: int32/uint32 [1] device counter, zero)."""
    B, P = status.shape
    _need_cuda(status, kf_member, counts, flag, done, totals, kf_count)
    _check(load().v2d_survival_decide(_p(status), _p(kf_member), B, P, _p(counts), float(T),
                                      _p(flag), _p(totals), _p(kf_count), int(cond_handle),
                                      _p(done), _stream()), "survival_decide")


def ring_tables(table, counter, cur, prev):
    """v2d_ring_tables: rows counter and counter-1 (mod R) of the [R, C] int64 device
    pointer table into cur / prev, then counter += 1 (all on the device)."""
    R, C = table.shape
    _need_cuda(table, counter, cur, prev)
    _check(load().v2d_ring_tables(_p(table), R, C, _p(counter), _p(cur), _p(prev), _stream()),
           "ring_tables")


def refill_tracks(kp_xy, cell_count, grid_x, grid_y, k, flag, tracks, status, kf_member,
                  track_id, next_id):
    B, P = status.shape
    _need_cuda(kp_xy, cell_count, flag, tracks, status, kf_member, track_id, next_id)
    _check(load().v2d_refill_tracks(_p(kp_xy), _p(cell_count), grid_x, grid_y, k, _p(flag), B, P,
                                    _p(tracks), _p(status), _p(kf_member), _p(track_id),
                                    _p(next_id), _stream()), "refill_tracks")
