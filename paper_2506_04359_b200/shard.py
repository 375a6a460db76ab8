"""Multi-GPU host logic: who processes which (camera, frame) units, and the
assembly of per-camera track lists across ranks.

Cameras are independent ("feature selection happens independently for each
camera") and, with re-detection every frame (DESIGN.md reading
#21), so are frame pairs; the only coupling is the previous frame's pyramid, so a
frame chunk starts one frame early.  Nothing in the data path needs a
collective; the one exchange is the rig-wide track list ("we collect all the
available observations ... for pose estimation"), gathered with
`all_gather_into_tensor` (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Shard:
    cams: tuple          # camera indices owned by this rank (contiguous block)
    frame_begin: int     # first frame whose tracks this rank produces
    frame_end: int       # one past the last
    prime_frame: int     # frame whose pyramid/keypoints are built first (frame_begin - 1, or -1)


def shard_plan(n_cams: int, n_frames: int, world: int, rank: int) -> Shard:
    """Strong-scaling partition of a fixed rig stream over `world` ranks.

    C >= G: contiguous camera blocks (keeps stereo pairs (2i, 2i+1) together
    when C/G is even), all frames.  C < G: each camera is shared by G/C ranks
    which split its frames into contiguous chunks; a chunk starts one frame early
    (prime_frame) to build the previous pyramid.  Requires C % G == 0 or
    G % C == 0."""
    if world < 1 or not (0 <= rank < world) or n_cams < 1 or n_frames < 2:
        raise ValueError("bad shard arguments")
    if n_cams >= world:
        if n_cams % world:
            raise ValueError("n_cams must be a multiple of world")
        per = n_cams // world
        return Shard(tuple(range(rank * per, (rank + 1) * per)), 1, n_frames, 0)
    if world % n_cams:
        raise ValueError("world must be a multiple of n_cams")
    per_cam = world // n_cams
    cam = rank // per_cam
    part = rank % per_cam
    # frames 1..n_frames-1 produce tracks (frame 0 only seeds keypoints)
    n_pairs = n_frames - 1
    b = 1 + part * n_pairs // per_cam
    e = 1 + (part + 1) * n_pairs // per_cam
    return Shard((cam,), b, e, b - 1)


class TrackGather:
    """All-gather of fixed-size per-step track lists: positions [B, P, 2] f32
    and statuses [B, P] u8 of every rank into [world*B, ...] tensors (rank-major).
    Buffers are allocated once; call `gather` on the stream that should carry
    the collective (the bench uses a side stream)."""

    def __init__(self, B: int, P: int, device, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.B, self.P = B, P
        self.all_pos = torch.empty((self.world * B, P, 2), dtype=torch.float32, device=device)
        self.all_status = torch.empty((self.world * B, P), dtype=torch.uint8, device=device)

    def gather(self, pos: torch.Tensor, status: torch.Tensor):
        if self.world == 1:
            self.all_pos.copy_(pos)
            self.all_status.copy_(status)
        else:
            dist.all_gather_into_tensor(self.all_pos, pos.contiguous(), group=self.group)
            dist.all_gather_into_tensor(self.all_status, status.contiguous(), group=self.group)
        return self.all_pos, self.all_status

    def rank_block(self, r: int):
        """Rank r's slice of the gathered lists."""
        return (self.all_pos[r * self.B:(r + 1) * self.B],
                self.all_status[r * self.B:(r + 1) * self.B])
