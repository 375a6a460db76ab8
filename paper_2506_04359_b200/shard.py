"""Multi-GPU host logic: who processes which (camera, frame) units, and the
assembly of per-camera track lists across ranks.

Cameras are independent ("feature selection happens independently for each
camera") and, with re-detection every frame (DESIGN.md reading
#21), so are frame pairs; the only coupling is the previous frame's pyramid, so a
frame chunk starts one frame early.  Nothing in the data path needs a
collective; the one exchange is the rig-wide track list ("we collect all the
available observations ... for pose estimation"): per-slot records
(x, y, status, ncc) written by the KLT kernel (v2d_track_klt's track_list,
SURVEY §8(a) a7), all-gathered with `all_gather_into_tensor` (NCCL on the GPU
box, gloo in the CPU tests and the one-GPU multi-rank tests), batched over
>= 16 frames per collective on a side stream.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

RECORD = 4  # (x, y, status, ncc) fp32 per track slot


@dataclass(frozen=True)
class Shard:
    cams: tuple          # camera indices owned by this rank (contiguous block)
    frame_begin: int     # first frame whose tracks this rank produces
    frame_end: int       # one past the last
    prime_frame: int     # frame whose pyramid/keypoints are built first (frame_begin - 1, or -1)


def shard_plan(n_cams: int, n_frames: int, world: int, rank: int) -> Shard:
    """Partition of a fixed rig stream of n_frames frames over `world` ranks.

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


@dataclass(frozen=True)
class RigShard:
    """The streams one rank processes in the ring bench: stream v is camera
    cams[v] starting at ring frame phases[v] (its first tracked frame; the
    frame before it is the chunk's prime frame)."""
    cams: tuple
    phases: tuple


def rig_shard(n_cams: int, ring: int, world: int, rank: int) -> RigShard:
    """shard_plan over a closed-loop ring of `ring` frames (the stream the bench
    loops over): camera blocks at phase 0 when C >= G; otherwise one camera per
    rank whose frames are split into G/C contiguous chunks, chunk p starting at
    ring frame p*ring/(G/C) (= shard_plan's prime_frame + 1 on a stream of
    ring + 1 frames).  `ring` must be a multiple of G/C."""
    sh = shard_plan(n_cams, ring + 1, world, rank)
    if n_cams >= world:
        return RigShard(sh.cams, (0,) * len(sh.cams))
    per_cam = world // n_cams
    if ring % per_cam:
        raise ValueError("ring must be a multiple of world / n_cams")
    return RigShard(sh.cams, (sh.frame_begin - 1,))


def all_streams(n_cams: int, ring: int, world: int) -> RigShard:
    """Every rank's streams in rank order (what one process must compute to
    reproduce the sharded run)."""
    cams, phases = [], []
    for r in range(world):
        s = rig_shard(n_cams, ring, world, r)
        cams += list(s.cams)
        phases += list(s.phases)
    return RigShard(tuple(cams), tuple(phases))


def _host_staged(group) -> bool:
    """gloo (the CPU tests and the one-GPU multi-rank tests) moves device
    tensors through host memory; NCCL reads device memory directly."""
    return dist.get_backend(group) == "gloo"


def all_gather_into(out: torch.Tensor, inp: torch.Tensor, group=None):
    """dist.all_gather_into_tensor on the current stream (rank-major), on flat
    views (out holds world * inp.numel() elements in rank order)."""
    flat_out = out.view(-1)
    if inp.is_cuda and _host_staged(group):
        h = torch.empty(flat_out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(h, inp.reshape(-1).cpu(), group=group)
        flat_out.copy_(h, non_blocking=False)
    else:
        dist.all_gather_into_tensor(flat_out, inp.contiguous().view(-1), group=group)


def all_reduce_sum_(t: torch.Tensor, group=None):
    """In-place dist.all_reduce(SUM) on the current stream."""
    if t.is_cuda and _host_staged(group):
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)


class TrackGather:
    """All-gather of fixed-size track-list records fp32 [n, P, 4] = (x, y,
    status, ncc) of every rank into [world*n, P, 4] (rank-major).  Buffers are
    allocated once; call `gather` on the stream that should carry the
    collective."""

    def __init__(self, n: int, P: int, device, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.n, self.P = n, P
        self.all = torch.empty((self.world * n, P, RECORD), dtype=torch.float32, device=device)

    def gather(self, records: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            self.all.copy_(records)
        else:
            all_gather_into(self.all, records, self.group)
        return self.all

    def rank_block(self, r: int) -> torch.Tensor:
        """Rank r's slice of the gathered records."""
        return self.all[r * self.n:(r + 1) * self.n]


class BatchedTrackGather:
    """Per-step track lists [B, P, 4] collected into a ring of `nb` steps and
    all-gathered once per `nb` steps (>= 16 frames per collective, SURVEY
    §8(e)) on a side stream, double-buffered so the KLT launches of the next
    batch overlap the collective of the previous one.

        recs = bg.slot(s)        # pass to v2d_track_klt as track_list
        ... launches of step s ...
        bg.step_done(s)          # every nb-th step: enqueue the gather
        bg.flush()               # current stream waits for every gather

    world == 1: no collective (the one rank already holds every list)."""

    def __init__(self, nb: int, B: int, P: int, device, group=None, side=None):
        self.nb, self.B, self.P = nb, B, P
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.local = torch.zeros((2, nb, B, P, RECORD), dtype=torch.float32, device=device)
        self.all = torch.zeros((2, self.world, nb, B, P, RECORD), dtype=torch.float32,
                               device=device)
        self.side = side if side is not None or self.world == 1 else torch.cuda.Stream(device)
        self.done = [None, None]
        self.n_gathers = 0

    def slot(self, s: int) -> torch.Tensor:
        h = (s // self.nb) % 2
        if s % self.nb == 0 and self.done[h] is not None:
            # the half is rewritten: its previous gather must have read it
            torch.cuda.current_stream().wait_event(self.done[h])
            self.done[h] = None
        return self.local[h, s % self.nb]

    def step_done(self, s: int):
        if self.world == 1 or (s + 1) % self.nb:
            return
        h = (s // self.nb) % 2
        ready = torch.cuda.Event()
        ready.record()
        with torch.cuda.stream(self.side):
            self.side.wait_event(ready)
            all_gather_into(self.all[h], self.local[h], self.group)
            ev = torch.cuda.Event()
            ev.record(self.side)
        self.done[h] = ev
        self.n_gathers += 1

    def flush_partial(self, s_last: int):
        """Gather the batch holding step s_last even if it is not full (end of
        a run); a full batch was already gathered by step_done."""
        if self.world == 1 or (s_last + 1) % self.nb == 0:
            return
        self.step_done(s_last + (self.nb - 1 - s_last % self.nb))

    def flush(self):
        for h in (0, 1):
            if self.done[h] is not None:
                torch.cuda.current_stream().wait_event(self.done[h])

    def gathered(self, s: int) -> torch.Tensor:
        """[world, B, P, 4] records of step s (valid after its batch's gather
        completed; world == 1: the local lists)."""
        h = (s // self.nb) % 2
        if self.world == 1:
            return self.local[h, s % self.nb][None]
        return self.all[h, :, s % self.nb]
