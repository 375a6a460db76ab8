"""Batched per-camera-frame pipeline over the C ABI.

One *step* processes F consecutive frames of C cameras (B = F*C images, batch
index b = f*C + c):

    v2d_build_pyramid(frames t..t+F-1)                      -> pyr[parity]
    v2d_detect_gftt  (frames t..t+F-1)                      -> kp slots 1..F
    v2d_track_klt    (pyr_{t+f-1} -> pyr_{t+f}, pts = kp slots 0..F-1)
    kp slot 0 <- kp slot F     (carry: frame t+F-1's keypoints feed the next step)

Frames are addressed through device pointer tables, so a ring of rendered
frames in HBM (bench `value`) and the three-slot staging buffers of HostStream,
filled from pinned host memory on a copy stream (bench `e2e`), run the same
three launches.  Nothing here computes
any part of the method: it allocates, builds pointer tables and calls the ABI.
"""
from __future__ import annotations

import torch

from . import vslam2d as v2d
from .vslam2d import FrontendConfig


class Frontend2D:
    """overlap=True: the KLT launch of the step's first frame (the C images whose
    keypoints were detected in the previous step) runs on a second stream,
    concurrently with the detection launch of this step — the two are
    independent (K2(t) needs frame t only, K3(t) needs the pyramids of t-1 and t
    and the keypoints of t-1), and their pipes are complementary (K2: integer alu
    pipe; K3: fma pipe and shared-memory loads).  The frames f >= 1 of a step
    (F > 1) are tracked after the detection launch, as before.  Results are
    identical (same kernels, same inputs)."""

    def __init__(self, cfg: FrontendConfig, cams: int, frames_per_step: int, device,
                 l0_pitch: int, overlap: bool = False):
        self.cfg, self.C, self.F, self.dev = cfg, cams, frames_per_step, torch.device(device)
        self.overlap = overlap
        if overlap:
            self.side = torch.cuda.Stream(device=self.dev)
            self.ev_pyr = torch.cuda.Event()
            self.ev_klt = torch.cuda.Event()
        self.B = cams * frames_per_step
        self.pitch = l0_pitch
        self.layout = v2d.pyramid_layout(cfg.W, cfg.H, cfg.levels)
        self.k = v2d.grid_k(cfg.grid_x, cfg.grid_y, cfg.k, cfg.K_min)
        self.P = cfg.grid_x * cfg.grid_y * self.k
        n = max(int(self.layout.floats_per_image), 32)
        d = self.dev
        # pyramids: two halves (step parity) x B images
        self.pyr = torch.zeros((2, self.B, n), dtype=torch.float32, device=d)
        # keypoints: slot j <-> frame t-1+j, each [C, P, 2] (batch order f*C + c)
        self.kp_xy = torch.full((frames_per_step + 1, cams, self.P, 2), -1.0,
                                dtype=torch.float32, device=d)
        self.kp_score = torch.zeros((frames_per_step + 1, cams, self.P), dtype=torch.float32,
                                    device=d)
        self.cell_count = torch.zeros((frames_per_step + 1, cams, cfg.grid_x * cfg.grid_y),
                                      dtype=torch.int32, device=d)
        self.pos = torch.zeros((self.B, self.P, 2), dtype=torch.float32, device=d)
        self.status = torch.zeros((self.B, self.P), dtype=torch.uint8, device=d)
        self.ncc = torch.zeros((self.B, self.P), dtype=torch.float32, device=d)
        self.iters = torch.zeros((self.B, self.P), dtype=torch.int32, device=d)
        # K2 workspace (dense two-pass detection): B*H*W floats
        self.ws = torch.empty((self.B, cfg.H, v2d.workspace_pitch(cfg.W)), dtype=torch.float32,
                              device=d)
        # pyramid pointer tables per parity: current and previous images (host
        # arithmetic, one H2D copy each)
        stride = self.pyr.stride(1) * 4
        addr = [[self.pyr[par].data_ptr() + i * stride for i in range(self.B)] for par in (0, 1)]
        cur, prev = [], []
        for par in (0, 1):
            # frame f-1 of this step; for f = 0, the last frame of the previous step
            pv = addr[1 - par][-cams:] + addr[par][:-cams]
            cur.append(v2d.ptr_table(addr[par], d))
            prev.append(v2d.ptr_table(pv, d))
        self.pyr_ptrs, self.prev_pyr_ptrs = cur, prev
        # our kernels per step: pyramid, GFTT pass A + pass B (workspace path), KLT
        self.launches_per_step = 4

    # ------------------------------------------------------------------
    def step(self, l0_ptrs: torch.Tensor, prev_l0_ptrs: torch.Tensor, parity: int,
             status_out: torch.Tensor | None = None, events=None,
             track_list: torch.Tensor | None = None):
        """Enqueue one step.  l0_ptrs / prev_l0_ptrs: device int64 [B] pointer
        tables of frames t+f and t+f-1 (batch order f*C + c).  `events`
        (optional, 4 CUDA events) bracket the three launches for per-kernel
        timing on the launching stream.  `track_list` (optional fp32 [B, P, 4])
        receives the step's (x, y, status, ncc) records from the KLT kernel
        (SURVEY §8(a) a7)."""
        c, B = self.cfg, self.B
        W, H, L = c.W, c.H, c.levels
        st = self.status if status_out is None else status_out

        def klt(lo, hi):  # images [lo, hi) of the step (frames lo/C .. hi/C - 1)
            if hi <= lo:
                return
            v2d.track_klt_ptrs(prev_l0_ptrs[lo:hi], self.prev_pyr_ptrs[parity][lo:hi],
                               l0_ptrs[lo:hi], self.pyr_ptrs[parity][lo:hi], self.pitch, hi - lo,
                               W, H, L, self.kp_xy[:-1].reshape(B, self.P, 2)[lo:hi], None, None,
                               self.P, c.win, c.iters, c.eps, c.ncc_min, c.min_eig,
                               self.pos[lo:hi], st[lo:hi], self.ncc[lo:hi], self.iters[lo:hi],
                               c.klt_flags, None if track_list is None else track_list[lo:hi])

        if events is not None:
            events[0].record()
        v2d.build_pyramid_ptrs(l0_ptrs, self.pitch, B, W, H, L, self.pyr_ptrs[parity])
        if events is not None:
            events[1].record()
        if self.overlap:
            main = torch.cuda.current_stream()
            self.ev_pyr.record(main)
            with torch.cuda.stream(self.side):
                self.side.wait_event(self.ev_pyr)
                klt(0, self.C)
                self.ev_klt.record(self.side)
        v2d.detect_gftt_ptrs(l0_ptrs, self.pitch, B, W, H, c.grid_x, c.grid_y, c.k, c.K_min,
                             c.min_score, c.border, c.nms, self.kp_xy[1:], self.kp_score[1:],
                             self.cell_count[1:], workspace=self.ws)
        if events is not None:
            events[2].record()
        if self.overlap:
            klt(self.C, B)
            torch.cuda.current_stream().wait_event(self.ev_klt)
        else:
            klt(0, B)
        if events is not None:
            events[3].record()
        self.kp_xy[0].copy_(self.kp_xy[-1], non_blocking=True)

    def prime(self, l0_ptrs_last: torch.Tensor, parity_prev: int):
        """Fill the previous-frame state (pyramid of the frame before the first
        step, and its keypoints) so step 0 tracks real data."""
        c = self.cfg
        C = self.C
        pyr_ptrs = self.pyr_ptrs[parity_prev][-C:]
        v2d.build_pyramid_ptrs(l0_ptrs_last, self.pitch, C, c.W, c.H, c.levels, pyr_ptrs)
        v2d.detect_gftt_ptrs(l0_ptrs_last, self.pitch, C, c.W, c.H, c.grid_x, c.grid_y, c.k,
                             c.K_min, c.min_score, c.border, c.nms, self.kp_xy[0],
                             self.kp_score[0], self.cell_count[0], workspace=self.ws)


class HostStream:
    """Public streaming entry point for frames that live in (pinned) host memory.

    Per step s the caller hands in the host batch of step s+1 and gets back the
    host results of step s:

        copy stream : wait kernels(s-1) -> H2D frames(s+1) into slot (s+1) % 3
        main stream : wait H2D(s) -> the three launches of step s -> snapshot
                      (D2D) of the step's keypoints, positions and statuses
        read stream : wait kernels(s) -> D2H of the snapshot into pinned buffers

    so uploads and read-backs overlap the kernels.  The read-backs have their own
    stream (the other copy direction): on one stream a read-back waiting for step s's
    kernels held back the upload of step s+2 queued behind it.  Three device frame slots are
    needed because step s reads its own frames and the last frame of step s-1;
    two snapshot/host result sets let read-back s overlap kernels s+1."""

    def __init__(self, fe: Frontend2D):
        self.fe = fe
        B, C, P, F = fe.B, fe.C, fe.P, fe.F
        d = fe.dev
        self.dbuf = torch.empty((3, B, fe.cfg.H, fe.pitch), dtype=torch.uint8, device=d)
        stride = self.dbuf.stride(1)
        addr = [[self.dbuf[i].data_ptr() + b * stride for b in range(B)] for i in range(3)]
        self.cur_t = [v2d.ptr_table(addr[i], d) for i in range(3)]
        # previous frame of batch entry f*C + c: entry (f-1)*C + c, or for f = 0 the
        # last frame of the slot before
        self.prev_t = [v2d.ptr_table(addr[(i - 1) % 3][-C:] + addr[i][:-C], d) for i in range(3)]
        self.copy = torch.cuda.Stream(device=d)
        self.read = torch.cuda.Stream(device=d)
        self.ev_in = [torch.cuda.Event() for _ in range(3)]
        self.ev_done = [torch.cuda.Event() for _ in range(3)]
        self.ev_out = [torch.cuda.Event() for _ in range(2)]
        self.snap_kp = torch.empty((2, F, C, P, 2), dtype=torch.float32, device=d)
        self.snap_pos = torch.empty((2, B, P, 2), dtype=torch.float32, device=d)
        self.snap_st = torch.empty((2, B, P), dtype=torch.uint8, device=d)
        self.host_kp = torch.empty((2, F, C, P, 2), dtype=torch.float32, pin_memory=True)
        self.host_pos = torch.empty((2, B, P, 2), dtype=torch.float32, pin_memory=True)
        self.host_st = torch.empty((2, B, P), dtype=torch.uint8, pin_memory=True)
        self.h2d_bytes_per_step = B * fe.cfg.H * fe.pitch
        self.d2h_bytes_per_step = (self.host_kp[0].numel() * 4 + self.host_pos[0].numel() * 4 +
                                   self.host_st[0].numel())

    def upload(self, s: int, host_frames: torch.Tensor):
        """Enqueue the H2D copy of step s's frames (pinned [B, H, pitch] u8)."""
        k = s % 3
        with torch.cuda.stream(self.copy):
            if s >= 1:  # slot k was read by step s-3 (current) and s-2 (previous frame)
                self.copy.wait_event(self.ev_done[(s - 2) % 3])
            self.dbuf[k].copy_(host_frames, non_blocking=True)
            self.ev_in[k].record(self.copy)

    def start(self, host_frames_prev: torch.Tensor):
        """Prime with the batch preceding step 0 (its last C frames are used)."""
        fe = self.fe
        with torch.cuda.stream(self.copy):
            self.dbuf[2].copy_(host_frames_prev, non_blocking=True)
            self.ev_in[2].record(self.copy)
        torch.cuda.current_stream().wait_event(self.ev_in[2])
        fe.prime(self.cur_t[2][-fe.C:], 1)
        self.ev_done[2].record()
        self.ev_done[1].record()

    def compute(self, s: int):
        """Enqueue step s's kernels (after its upload) and its result snapshot."""
        fe, k, j = self.fe, s % 3, s % 2
        cs = torch.cuda.current_stream()
        cs.wait_event(self.ev_in[k])
        fe.step(self.cur_t[k], self.prev_t[k], j)
        if s >= 2:  # snapshot j is free once read-back s-2 is done
            cs.wait_event(self.ev_out[j])
        self.snap_kp[j].copy_(fe.kp_xy[1:], non_blocking=True)
        self.snap_pos[j].copy_(fe.pos, non_blocking=True)
        self.snap_st[j].copy_(fe.status, non_blocking=True)
        self.ev_done[k].record(cs)

    def download(self, s: int):
        """Enqueue the D2H read-back of step s's results into host set s % 2."""
        j = s % 2
        with torch.cuda.stream(self.read):
            self.read.wait_event(self.ev_done[s % 3])
            self.host_kp[j].copy_(self.snap_kp[j], non_blocking=True)
            self.host_pos[j].copy_(self.snap_pos[j], non_blocking=True)
            self.host_st[j].copy_(self.snap_st[j], non_blocking=True)
            self.ev_out[j].record(self.read)

    def results(self, s: int):
        """Host (kp_xy, pos, status) of step s once ev_out[s % 2] has completed."""
        self.ev_out[s % 2].synchronize()
        j = s % 2
        return self.host_kp[j], self.host_pos[j], self.host_st[j]

    def finish(self):
        """Make the main stream wait for all pending copies."""
        torch.cuda.current_stream().wait_stream(self.copy)
        torch.cuda.current_stream().wait_stream(self.read)


class RingSchedule:
    """Pointer tables for stepping through a device ring frames[C, R, H, pitch]
    F frames at a time (R must be a multiple of 2F so parity and ring index
    advance together).

    `cams` / `phases` (optional, one entry per processed stream v) select the
    ring camera of stream v and the ring frame it starts at: step s, frame f of
    stream v is ring frame (phases[v] + s*F + f) mod R of camera cams[v] (batch
    entry f*V + v), and `before_first[v]` is the frame before its start.  The
    multi-GPU shards (shard.rig_shard) are such streams: a block of cameras at
    phase 0, or one camera's frame chunk starting at its phase."""

    def __init__(self, frames: torch.Tensor, F: int, cams=None, phases=None):
        Cr, R = frames.shape[0], frames.shape[1]
        assert R % (2 * F) == 0, "ring length must be a multiple of 2F"
        cams = list(range(Cr)) if cams is None else [int(c) for c in cams]
        phases = [0] * len(cams) if phases is None else [int(p) for p in phases]
        assert len(phases) == len(cams) and all(0 <= c < Cr for c in cams)
        C = len(cams)
        self.C, self.R, self.F = C, R, F
        self.cams, self.phases = cams, phases
        self.n_steps = R // F
        img = frames.stride(1) * frames.element_size()
        cam = frames.stride(0) * frames.element_size()
        base = frames.data_ptr()
        dev = frames.device
        addr = lambda v, t: base + cams[v] * cam + ((phases[v] + t) % R) * img
        cur = [[addr(v, s * F + f) for f in range(F) for v in range(C)]
               for s in range(self.n_steps)]
        prev = [[addr(v, s * F + f - 1) for f in range(F) for v in range(C)]
                for s in range(self.n_steps)]
        self.cur = torch.tensor(cur, dtype=torch.int64).to(dev)      # [n_steps, F*C]
        self.prev = torch.tensor(prev, dtype=torch.int64).to(dev)
        self.before_first = v2d.ptr_table([addr(v, -1) for v in range(C)], dev)

    def tables(self, step: int):
        i = step % self.n_steps
        return self.cur[i], self.prev[i], i % 2


class KeyframeTracker:
    """Variant f1: keyframe-driven continuous tracking of one
    rig, one frame per step (B = C cameras).  Per frame:

        v2d_build_pyramid   (frame t)
        v2d_track_klt       (live tracks t-1 -> t; lost slots are SKIPPED because the
                             status table is fed back as in_status: lost is terminal)
        v2d_survival_decide (per camera |S_kf|, |S_curr ∩ S_kf| and the rig-wide Eq. 5
                             decision into a device flag, one launch; multi-GPU:
                             v2d_track_survival, an all-reduce of the totals, then
                             v2d_keyframe_decide)
        -- device-flag gated, no host round trip --
        v2d_suppress_mask   (min_separation disks around live tracks)
        v2d_detect_gftt     (masked grid top-k)
        v2d_refill_tracks   (new tracks into dead slots, new ids; S_kf := alive)

    The track table is double-buffered: KLT reads table i and writes table 1-i.
    """

    def __init__(self, cfg: FrontendConfig, cams: int, device, l0_pitch: int, T: float = 0.7,
                 min_sep: float | None = None, group=None):
        self.cfg, self.C, self.dev, self.pitch = cfg, cams, torch.device(device), l0_pitch
        self.T = T
        self.min_sep = float(cfg.win // 2 if min_sep is None else min_sep)
        self.group = group
        self.layout = v2d.pyramid_layout(cfg.W, cfg.H, cfg.levels)
        self.k = v2d.grid_k(cfg.grid_x, cfg.grid_y, cfg.k, cfg.K_min)
        self.P = cfg.grid_x * cfg.grid_y * self.k
        C, P, d = cams, self.P, self.dev
        n = max(int(self.layout.floats_per_image), 32)
        self.pyr = torch.zeros((2, C, n), dtype=torch.float32, device=d)
        self.pyr_ptrs = [v2d.ptrs_of(self.pyr[i]) for i in range(2)]
        self.tracks = torch.full((2, C, P, 2), -1.0, dtype=torch.float32, device=d)
        self.status = torch.full((2, C, P), v2d.SKIPPED, dtype=torch.uint8, device=d)
        self.kf_member = torch.zeros((C, P), dtype=torch.uint8, device=d)
        self.track_id = torch.full((C, P), -1, dtype=torch.int32, device=d)
        self.next_id = torch.zeros((C,), dtype=torch.int32, device=d)
        self.mask = torch.zeros((C, cfg.H, l0_pitch), dtype=torch.uint8, device=d)
        self.ws = torch.empty((C, cfg.H, v2d.workspace_pitch(cfg.W)), dtype=torch.float32, device=d)
        self.mask_ptrs = v2d.ptrs_of(self.mask)
        self.kp_xy = torch.full((C, cfg.grid_y, cfg.grid_x, self.k, 2), -1.0, device=d)
        self.kp_score = torch.zeros((C, cfg.grid_y, cfg.grid_x, self.k), device=d)
        self.cell_count = torch.zeros((C, cfg.grid_x * cfg.grid_y), dtype=torch.int32, device=d)
        self.counts = torch.zeros((C, 2), dtype=torch.int32, device=d)
        self.flag = torch.zeros((1,), dtype=torch.int32, device=d)
        self.totals = torch.zeros((2,), dtype=torch.int64, device=d)
        self.ncc = torch.zeros((C, P), device=d)
        self.iters = torch.zeros((C, P), dtype=torch.int32, device=d)
        self.kf_count = torch.zeros((), dtype=torch.int64, device=d)  # keyframes so far
        self.done = torch.zeros((1,), dtype=torch.int32, device=d)    # survival_decide counter
        self.cur = 0

    def _keyframe_branch(self, l0_ptrs, j):
        c, C, P = self.cfg, self.C, self.P
        v2d.suppress_mask_ptrs(self.tracks[j], self.status[j], C, P, self.min_sep, c.W, c.H,
                               self.mask_ptrs, self.pitch, self.flag)
        v2d.detect_gftt_ptrs(l0_ptrs, self.pitch, C, c.W, c.H, c.grid_x, c.grid_y, c.k, c.K_min,
                             c.min_score, c.border, c.nms, self.kp_xy, self.kp_score,
                             self.cell_count, None, self.mask_ptrs, self.flag, self.ws)
        v2d.refill_tracks(self.kp_xy, self.cell_count, c.grid_x, c.grid_y, self.k, self.flag,
                          self.tracks[j], self.status[j], self.kf_member, self.track_id,
                          self.next_id)

    def start(self, l0_ptrs: torch.Tensor):
        """First frame: pyramid + bootstrap keyframe (Eq. 5 with empty S_kf)."""
        c = self.cfg
        v2d.build_pyramid_ptrs(l0_ptrs, self.pitch, self.C, c.W, c.H, c.levels,
                               self.pyr_ptrs[self.cur])
        self.flag.fill_(1)
        self._keyframe_branch(l0_ptrs, self.cur)

    def step(self, l0_ptrs: torch.Tensor, prev_l0_ptrs: torch.Tensor):
        c, C, P = self.cfg, self.C, self.P
        i, j = self.cur, 1 - self.cur
        v2d.build_pyramid_ptrs(l0_ptrs, self.pitch, C, c.W, c.H, c.levels, self.pyr_ptrs[j])
        v2d.track_klt_ptrs(prev_l0_ptrs, self.pyr_ptrs[i], l0_ptrs, self.pyr_ptrs[j], self.pitch,
                           C, c.W, c.H, c.levels, self.tracks[i], None, self.status[i], P, c.win,
                           c.iters, c.eps, c.ncc_min, c.min_eig, self.tracks[j], self.status[j],
                           self.ncc, self.iters, c.klt_flags)
        if self.group is None:  # one launch: counts and the rig-wide Eq. 5 decision
            v2d.survival_decide(self.status[j], self.kf_member, self.counts, self.T, self.flag,
                                self.done, self.totals)
            self._keyframe_branch(l0_ptrs, j)
            self.cur = j
            return
        v2d.track_survival(self.status[j], self.kf_member, self.counts)
        if self.group is not None:
            from .shard import all_reduce_sum_
            v2d.keyframe_decide(self.counts, self.T, self.flag, self.totals)
            all_reduce_sum_(self.totals, self.group)  # rig-wide Eq. 5 (NCCL)
            red = self.totals.to(torch.int32).view(1, 2)
            v2d.keyframe_decide(red, self.T, self.flag)
        else:
            v2d.keyframe_decide(self.counts, self.T, self.flag, self.totals)
        self._keyframe_branch(l0_ptrs, j)
        self.cur = j

    # ------------------------------------------------------------ CUDA graphs
    def _main(self, l0_ptrs, prev_l0_ptrs, j, cond_handle=0):
        """The unconditional part of a frame (pyramid, KLT, survival, decide)."""
        c, C, P = self.cfg, self.C, self.P
        i = 1 - j
        v2d.build_pyramid_ptrs(l0_ptrs, self.pitch, C, c.W, c.H, c.levels, self.pyr_ptrs[j])
        v2d.track_klt_ptrs(prev_l0_ptrs, self.pyr_ptrs[i], l0_ptrs, self.pyr_ptrs[j], self.pitch,
                           C, c.W, c.H, c.levels, self.tracks[i], None, self.status[i], P, c.win,
                           c.iters, c.eps, c.ncc_min, c.min_eig, self.tracks[j], self.status[j],
                           self.ncc, self.iters, c.klt_flags)
        v2d.survival_decide(self.status[j], self.kf_member, self.counts, self.T, self.flag,
                            self.done, self.totals, self.kf_count, cond_handle)

    def capture(self, frame_table: torch.Tensor, next_frame: int, conditional: bool = True):
        """Record the per-frame step as CUDA graphs (the loop is launch-bound: 8+
        small launches per rig-frame).  frame_table: device int64 [R, C] frame
        pointers, frame t = row t % R; next_frame: index of the next frame to
        process.  The frame tables come from a device frame counter (v2d_ring_tables),
        so replay() needs no host work besides one graph launch; one graph per
        track-table parity.  conditional=True (default) builds each graph with the
        CUDA graph API (cuda-python): the keyframe branch is the body of an IF node
        whose value the decide kernel sets (v2d_keyframe_decide_graph), so a
        non-keyframe frame runs 5 kernels and no empty grids; conditional=False (or
        no conditional-node support) captures with torch.cuda.graph, the branch's
        kernels exiting on the device flag.  Single-process only (group is None)."""
        assert self.group is None, "graph capture of the multi-GPU all-reduce is not supported"
        self._ft = frame_table.contiguous()
        self._t = torch.full((1,), next_frame, dtype=torch.int64, device=self.dev)
        self._l0 = torch.empty((self.C,), dtype=torch.int64, device=self.dev)
        self._pl0 = torch.empty((self.C,), dtype=torch.int64, device=self.dev)
        torch.cuda.synchronize(self.dev)
        self._graphs, self._execs = {}, {}
        cur0 = self.cur
        self.graph_kind = "torch"
        if conditional:
            try:
                for par in (cur0, 1 - cur0):
                    self._execs[par] = self._capture_conditional(1 - par)
                self.graph_kind = "conditional"
            except Exception as e:  # no conditional nodes (driver / cuda-python): fallback
                self._execs = {}
                self.graph_fallback_reason = f"{type(e).__name__}: {e}"
        if not self._execs:
            for par in (cur0, 1 - cur0):
                j = 1 - par
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    v2d.ring_tables(self._ft, self._t, self._l0, self._pl0)
                    self._main(self._l0, self._pl0, j)
                    self._keyframe_branch(self._l0, j)
                self._graphs[par] = g
        self.cur = cur0
        torch.cuda.synchronize(self.dev)

    def _capture_conditional(self, j):
        """One frame (parity: KLT writes table j) as a CUDA graph whose keyframe branch
        is the body of a conditional IF node: ring tables -> pyramid -> KLT ->
        survival -> decide (sets the node's value) -> IF(flag){suppress, detect,
        refill}."""
        from cuda.bindings import runtime as rt

        def ok(r):  # cuda-python returns (err, *outputs)
            r = r if isinstance(r, tuple) else (r,)
            if r[0] != rt.cudaError_t.cudaSuccess:
                raise RuntimeError(f"CUDA graph API: {r[0]}")
            return None if len(r) == 1 else (r[1] if len(r) == 2 else r[1:])

        graph = ok(rt.cudaGraphCreate(0))
        handle = ok(rt.cudaGraphConditionalHandleCreate(graph, 0, 0))
        s = torch.cuda.Stream(self.dev)
        mode = rt.cudaStreamCaptureMode.cudaStreamCaptureModeThreadLocal
        with torch.cuda.stream(s):
            ok(rt.cudaStreamBeginCaptureToGraph(s.cuda_stream, graph, None, None, 0, mode))
            v2d.ring_tables(self._ft, self._t, self._l0, self._pl0)
            self._main(self._l0, self._pl0, j, int(handle))
            ok(rt.cudaStreamEndCapture(s.cuda_stream))
        # the captured main part is a chain: its one leaf node precedes the IF node
        nodes, n = ok(rt.cudaGraphGetNodes(graph, 0))
        nodes, n = ok(rt.cudaGraphGetNodes(graph, n))
        leaves = [nd for nd in nodes if ok(rt.cudaGraphNodeGetDependentNodes(nd, 0))[1] == 0]
        assert len(leaves) == 1, len(leaves)
        params = rt.cudaGraphNodeParams()
        params.type = rt.cudaGraphNodeType.cudaGraphNodeTypeConditional
        params.conditional.handle = handle
        params.conditional.type = rt.cudaGraphConditionalNodeType.cudaGraphCondTypeIf
        params.conditional.size = 1
        ok(rt.cudaGraphAddNode(graph, leaves, 1, params))
        body = params.conditional.phGraph_out[0]
        with torch.cuda.stream(s):
            ok(rt.cudaStreamBeginCaptureToGraph(s.cuda_stream, body, None, None, 0, mode))
            self._keyframe_branch(self._l0, j)
            ok(rt.cudaStreamEndCapture(s.cuda_stream))
        exe = ok(rt.cudaGraphInstantiate(graph, 0))
        self._cuda_graphs = getattr(self, "_cuda_graphs", []) + [graph]  # keep alive
        return exe

    def replay(self):
        """One rig-frame through the captured graph of the current parity."""
        if self._execs:
            from cuda.bindings import runtime as rt
            err = rt.cudaGraphLaunch(self._execs[self.cur],
                                     torch.cuda.current_stream(self.dev).cuda_stream)
            err = err[0] if isinstance(err, tuple) else err
            if err != rt.cudaError_t.cudaSuccess:
                raise RuntimeError(f"cudaGraphLaunch: {err}")
        else:
            self._graphs[self.cur].replay()
        self.cur = 1 - self.cur

    def table(self):
        """(tracks [C,P,2], status [C,P], kf_member, track_id, next_id) of the current frame."""
        return (self.tracks[self.cur], self.status[self.cur], self.kf_member, self.track_id,
                self.next_id)
