"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

This module holds NO arithmetic of the method (no pyramid, gradient, response,
selection or tracking): it only renders u8 frame streams with known sub-pixel
motion, so that the CUDA path and the oracle can be fed the same bytes
(task rule ③: "only the seeded input generators serve both").

Recipe (SURVEY.md §8(d) "Synthetic inputs", restated in DESIGN.md §4):
  * world texture per camera: white noise blurred at sigma 1.5, 3, 6 px
    (weights 1, 0.6, 0.4), rescaled to mean 128 / std 40, plus ~200 random
    uniform-gray rectangles (8-64 px) per Mpx for strong corners;
  * frame t = round-half-even(clamp(Catmull-Rom sample of the texture at
    (x - o_t.x, y - o_t.y), 0, 255)), so the true displacement of frame t-1 -> t
    is o_t - o_{t-1};
  * o_t is a closed loop with period R = ring length, so a ring wraps
    seamlessly; each camera has its own seeded phase (independent motion);
  * seeds: 0x250604359 ^ (cfg << 40) ^ (camera << 20).
Everything runs through torch so that the bench can render its rings in HBM;
noise and rectangle parameters are drawn with numpy PCG64 on the host, so the
stream is identical in distribution on every device (bytes can differ between
CPU and GPU rendering by rounding; parity tests always feed both sides the same
bytes).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

BASE_SEED = 0x250604359


def seed_for(cfg_index: int, camera: int, extra: int = 0) -> int:
    return (BASE_SEED ^ (cfg_index << 40) ^ (camera << 20) ^ extra) & ((1 << 63) - 1)


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


# --------------------------------------------------------------------------
# Workloads (BASELINE.json configs; unstated parameters are SURVEY §8(d)'s
# proposal).  Pure data: sizes and knobs, no method arithmetic.
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Workload:
    name: str
    index: int
    W: int
    H: int
    cams: int
    levels: int
    grid_x: int = 8
    grid_y: int = 8
    K_min: int = 0
    k: int = 0           # 0 -> Eq. 1 rule
    win: int = 21
    iters: int = 10
    eps: float = 0.01
    ncc_min: float = 0.8
    min_eig: float = 0.01
    motion: tuple = (6.0, 0.0)    # max per-frame |dx|, |dy| (px)
    frames: int = 1000
    fixed_motion: tuple | None = None
    stereo_disparity: float = 20.0  # odd camera = even camera's plane seen 20 px to the left
    description: str = ""

    @property
    def border(self) -> int:
        return (self.win - 1) // 2 + 1

    @property
    def pitch(self) -> int:
        return round_up(self.W, 64)


WORKLOADS = {
    "c1": Workload("c1", 0, 640, 480, 1, 3, K_min=200, k=4, frames=2,
                   fixed_motion=(3.2, -1.7),
                   description="single synthetic 640x480 grayscale frame pair, 3-level pyramid, "
                               "8x8 grid, k=4, 21x21 KLT window"),
    "c2": Workload("c2", 1, 752, 480, 2, 4, K_min=1000, motion=(4.24, 4.24), frames=1000,
                   description="EuRoC-shaped stereo stream 752x480 x2 cameras, 4-level pyramid, "
                               "~1000 keypoints/frame"),
    "c3": Workload("c3", 2, 1241, 376, 2, 4, K_min=2000, motion=(11.5, 3.0), frames=4500,
                   description="KITTI-shaped stereo stream 1241x376 x2 cameras, 4-level pyramid, "
                               "~2000 keypoints/frame"),
    "c4": Workload("c4", 3, 1280, 720, 8, 4, K_min=1500, motion=(5.6, 5.6), frames=1000,
                   description="multi-stereo rig 4 stereo pairs (8 cameras) 1280x720, "
                               "~1500 keypoints/camera"),
    "c5": Workload("c5", 4, 1920, 1200, 32, 5, K_min=2000, motion=(5.6, 5.6), frames=1000,
                   description="32-camera rig 1920x1200, 5-level pyramid, ~2000 keypoints/camera"),
}


# --------------------------------------------------------------------------
# Texture
# --------------------------------------------------------------------------
def _gauss_taps(sigma: float) -> torch.Tensor:
    r = int(math.ceil(3 * sigma))
    x = torch.arange(-r, r + 1, dtype=torch.float64)
    g = torch.exp(-0.5 * (x / sigma) ** 2)
    return (g / g.sum()).float()


def _blur(img: torch.Tensor, sigma: float) -> torch.Tensor:
    """Separable Gaussian blur with reflect padding. img: [h, w] float32."""
    taps = _gauss_taps(sigma).to(img.device)
    r = taps.numel() // 2
    x = img[None, None]
    x = torch.nn.functional.pad(x, (r, r, 0, 0), mode="reflect")
    x = torch.nn.functional.conv2d(x, taps.view(1, 1, 1, -1))
    x = torch.nn.functional.pad(x, (0, 0, r, r), mode="reflect")
    x = torch.nn.functional.conv2d(x, taps.view(1, 1, -1, 1))
    return x[0, 0]


DEFAULT_OCTAVES = ((1.5, 1.0), (3.0, 0.6), (6.0, 0.4))
SMOOTH_OCTAVES = ((3.0, 0.6), (6.0, 0.4))


def make_texture(h: int, w: int, seed: int, device="cpu", rects_per_mpx: float = 200.0,
                 smooth: bool = False, octaves=None) -> torch.Tensor:
    """World texture [h, w] float32 (values roughly 0..255).  `octaves` is a
    list of (sigma, weight) blur scales; smooth=True drops the finest octave
    and the rectangles."""
    rng = np.random.Generator(np.random.PCG64(seed))
    noise = torch.from_numpy(rng.standard_normal((h, w), dtype=np.float32)).to(device)
    octaves = octaves or (SMOOTH_OCTAVES if smooth else DEFAULT_OCTAVES)
    tex = sum(wt * _blur(noise, sg) for sg, wt in octaves)
    tex = (tex - tex.mean()) / (tex.std() + 1e-12) * 40.0 + 128.0
    if not smooth:
        n_rect = int(round(rects_per_mpx * h * w / 1e6))
        ys = rng.integers(0, h, n_rect)
        xs = rng.integers(0, w, n_rect)
        hs = rng.integers(8, 65, n_rect)
        ws = rng.integers(8, 65, n_rect)
        gs = rng.uniform(10.0, 245.0, n_rect)
        for i in range(n_rect):
            tex[ys[i]:ys[i] + hs[i], xs[i]:xs[i] + ws[i]] = float(gs[i])
    return tex


# --------------------------------------------------------------------------
# Trajectory (closed loop) and rendering
# --------------------------------------------------------------------------
def trajectory(R: int, motion: tuple, seed: int) -> np.ndarray:
    """o_t, t = 0..R-1, float64 [R, 2]; |o_t - o_{t-1}| <= motion per axis,
    periodic with period R (o_R == o_0)."""
    rng = np.random.Generator(np.random.PCG64(seed ^ 0x7F4A7C15))
    phx, phy = rng.uniform(0, 2 * math.pi, 2)
    mx, my = motion
    ax = mx * R / (2 * math.pi)
    ay = my * R / (4 * math.pi)
    t = np.arange(R, dtype=np.float64)
    th = 2 * math.pi * t / R
    return np.stack([ax * np.sin(th + phx), ay * np.sin(2 * th + phy)], axis=1)


def _catmull_rom_weights(f: float) -> list[float]:
    f2, f3 = f * f, f * f * f
    return [(-f3 + 2 * f2 - f) / 2, (3 * f3 - 5 * f2 + 2) / 2, (-3 * f3 + 4 * f2 + f) / 2,
            (f3 - f2) / 2]


def render(tex: torch.Tensor, offsets: np.ndarray, H: int, W: int, pitch: int | None = None,
           origin: tuple[int, int] | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Frames [T, H, pitch] uint8 on tex.device: frame t (x, y) = tex sampled at
    (origin + (x, y) - o_t) with separable Catmull-Rom, rounded half-even and
    clamped to 0..255.  Columns >= W of each row are zero."""
    pitch = pitch or W
    th, tw = tex.shape
    ox0, oy0 = origin if origin is not None else ((tw - W) // 2, (th - H) // 2)
    T = offsets.shape[0]
    if out is None:
        out = torch.zeros((T, H, pitch), dtype=torch.uint8, device=tex.device)
    for t in range(T):
        sx = ox0 - float(offsets[t, 0])
        sy = oy0 - float(offsets[t, 1])
        ix, iy = math.floor(sx), math.floor(sy)
        wx, wy = _catmull_rom_weights(sx - ix), _catmull_rom_weights(sy - iy)
        if ix - 1 < 0 or iy - 1 < 0 or ix + W + 2 > tw or iy + H + 2 > th:
            raise ValueError("texture too small for the trajectory")
        rows = tex[iy - 1:iy + H + 2]
        hx = sum(wx[k] * rows[:, ix - 1 + k: ix - 1 + k + W] for k in range(4))
        v = sum(wy[k] * hx[k:k + H] for k in range(4))
        out[t, :, :W] = torch.round(v.clamp(0.0, 255.0)).to(torch.uint8)
    return out


@dataclass
class Stream:
    """A rendered per-camera frame ring: frames [cams, R, H, pitch] u8 and the
    true offsets [cams, R, 2] (true displacement t-1 -> t is o_t - o_{t-1})."""
    frames: torch.Tensor
    offsets: np.ndarray
    wl: Workload
    extra: dict = field(default_factory=dict)

    def true_displacement(self, cam: int, t: int) -> np.ndarray:
        R = self.offsets.shape[1]
        return self.offsets[cam, t % R] - self.offsets[cam, (t - 1) % R]


def make_stream(wl: Workload, ring: int, device="cpu", cams: list[int] | None = None,
                 rank_salt: int = 0, smooth: bool = False, only=None) -> Stream:
    """Render `ring` frames for each camera in `cams` (default all).  Cameras
    (2i, 2i+1) form rectified stereo pairs when wl.stereo_disparity > 0: the
    right camera renders the left camera's texture and trajectory shifted by the
    disparity (a fronto-parallel plane), so cross-camera tracking (f2) has a
    known answer; all other cameras are independent.  `only` (optional, a set of
    ring frame indices) renders just those frames of the same ring (the others
    stay zero): a camera's frame t depends only on (seed, camera, ring, t)."""
    cams = list(range(wl.cams)) if cams is None else cams
    frames = torch.zeros((len(cams), ring, wl.H, wl.pitch), dtype=torch.uint8, device=device)
    offs = np.zeros((len(cams), ring, 2))
    tex_cache = {}
    for ci, c in enumerate(cams):
        stereo_right = wl.stereo_disparity > 0 and (c % 2 == 1)
        src = c - 1 if stereo_right else c
        seed = seed_for(wl.index, src, rank_salt)
        if wl.fixed_motion is not None:
            o = np.zeros((ring, 2))
            for t in range(1, ring):
                o[t] = o[t - 1] + np.asarray(wl.fixed_motion)
        else:
            o = trajectory(ring, wl.motion, seed)
        disp = wl.stereo_disparity if wl.stereo_disparity > 0 else 0.0
        span_x = int(math.ceil(np.abs(o[:, 0]).max() + disp)) + 4
        span_y = int(math.ceil(np.abs(o[:, 1]).max())) + 4
        if src not in tex_cache:
            tex_cache[src] = make_texture(wl.H + 2 * span_y, wl.W + 2 * span_x, seed, device,
                                          smooth=smooth)
        tex = tex_cache[src]
        oo = o - np.array([disp, 0.0]) if stereo_right else o
        if only is None:
            render(tex, oo, wl.H, wl.W, wl.pitch, origin=(span_x, span_y), out=frames[ci])
        else:
            for t in sorted({int(t) % ring for t in only}):
                render(tex, oo[t:t + 1], wl.H, wl.W, wl.pitch, origin=(span_x, span_y),
                       out=frames[ci, t:t + 1])
        offs[ci] = oo
    return Stream(frames, offs, wl)


def noise_frame(H: int, W: int, seed: int) -> np.ndarray:
    """Independent uniform-noise u8 frame (for the NCC-rejection pin)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, 256, (H, W), dtype=np.uint8)


def shifted_pair(H: int, W: int, shift: tuple[float, float], seed: int, smooth: bool = False,
                 pitch: int | None = None):
    """Two u8 frames where frame 1 is frame 0 translated by `shift` (px)."""
    sx, sy = shift
    span = int(math.ceil(max(abs(sx), abs(sy)))) + 4
    tex = make_texture(H + 2 * span, W + 2 * span, seed, "cpu", smooth=smooth)
    o = np.array([[0.0, 0.0], [sx, sy]])
    fr = render(tex, o, H, W, pitch or W, origin=(span, span))
    return fr[0].numpy(), fr[1].numpy()


def stereo_pair(H: int, W: int, disparity: float, seed: int, smooth: bool = False,
                occluder: tuple | None = None, pitch: int | None = None):
    """Rectified stereo pair of a fronto-parallel textured plane: the right image
    sees world point x at x - disparity (disparity = fx * b / z; SPEC S:179 uses
    fx=400, b=0.1 m, z=2 m -> 20 px).  `occluder` = (x0, y0, w, h) paints a
    uniform block into the right image only."""
    left, right = shifted_pair(H, W, (-disparity, 0.0), seed, smooth=smooth, pitch=pitch)
    if occluder is not None:
        x0, y0, w, h = occluder
        right = right.copy()
        right[y0:y0 + h, x0:x0 + w] = 128
    return left, right
