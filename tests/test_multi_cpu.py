"""Multi-rank host logic on CPU (gloo, world_size 2): the shard plan covers every
(camera, frame) unit exactly once, and per-rank work assembled with the track
all-gather is bitwise identical to the single-process result.  Per-rank
compute is the oracle here (no GPU in this container); on the GPU box the same
TrackGather runs over NCCL inside bench.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2506_04359_b200.shard import (RECORD, TrackGather, all_streams, rig_shard,
                                          shard_plan)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("C,F,G", [(8, 10, 2), (8, 10, 4), (8, 10, 8), (2, 10, 4), (2, 11, 8),
                                   (32, 5, 8), (1, 9, 4)])
def test_shard_plan_partitions_units(C, F, G):
    seen = {}
    for r in range(G):
        sh = shard_plan(C, F, G, r)
        assert list(sh.cams) == list(range(sh.cams[0], sh.cams[-1] + 1))  # contiguous
        assert sh.prime_frame == sh.frame_begin - 1
        for c in sh.cams:
            for f in range(sh.frame_begin, sh.frame_end):
                assert (c, f) not in seen
                seen[(c, f)] = r
    assert set(seen) == {(c, f) for c in range(C) for f in range(1, F)}
    if C >= G and (C // G) % 2 == 0:
        for r in range(G):  # stereo pairs stay on one rank
            cams = shard_plan(C, F, G, r).cams
            assert all((c ^ 1) in cams for c in cams)


def test_shard_plan_rejects():
    with pytest.raises(ValueError):
        shard_plan(3, 10, 2, 0)
    with pytest.raises(ValueError):
        shard_plan(2, 10, 3, 0)


WL = synth.Workload("mt", 9, 160, 120, 2, 3, grid_x=2, grid_y=2, k=6, motion=(2.0, 1.5))
N_FRAMES = 5


def _frames():
    st = synth.make_stream(WL, N_FRAMES, "cpu")
    return st.frames[:, :, :, :WL.W].numpy().copy()


def _track_unit(frames, cam, f):
    """Oracle track-list records for frame pair (f-1 -> f) of camera cam:
    fp32 [P, 4] = (x, y, status, ncc)."""
    prev, cur = frames[cam, f - 1], frames[cam, f]
    _, dp = oracle.build_pyramid(prev, WL.levels)
    _, dc = oracle.build_pyramid(cur, WL.levels)
    xy, _, _ = oracle.detect_gftt(prev, WL.grid_x, WL.grid_y, k=WL.k, border=WL.border)
    pos, st, nc, _ = oracle.track_klt(dp, dc, WL.W, WL.H, WL.levels, xy.reshape(-1, 2),
                                      win=WL.win)
    return np.concatenate([pos, st[:, None], nc[:, None]], 1).astype(np.float32)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frames = _frames()
        sh = shard_plan(WL.cams, N_FRAMES, world, rank)
        units = [(c, f) for f in range(sh.frame_begin, sh.frame_end) for c in sh.cams]
        P = WL.grid_x * WL.grid_y * WL.k
        # fixed-size per-rank block: pad to the max units per rank
        n_max = max(len(shard_plan(WL.cams, N_FRAMES, world, r).cams) *
                    (shard_plan(WL.cams, N_FRAMES, world, r).frame_end -
                     shard_plan(WL.cams, N_FRAMES, world, r).frame_begin) for r in range(world))
        recs = torch.full((n_max, P, RECORD), -7.0)
        for i, (c, f) in enumerate(units):
            recs[i] = torch.from_numpy(_track_unit(frames, c, f))
        tg = TrackGather(n_max, P, "cpu")
        tg.gather(recs)
        if rank == 0:
            out = {}
            for r in range(world):
                shr = shard_plan(WL.cams, N_FRAMES, world, r)
                ur = [(c, f) for f in range(shr.frame_begin, shr.frame_end) for c in shr.cams]
                br = tg.rank_block(r)
                for i, u in enumerate(ur):
                    out[u] = br[i].numpy().copy()
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_equals_single(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    frames = _frames()
    assert set(out) == {(c, f) for c in range(WL.cams) for f in range(1, N_FRAMES)}
    for (c, f), rec in out.items():
        assert np.array_equal(rec, _track_unit(frames, c, f))


def test_track_gather_single_rank_identity():
    tg = TrackGather(3, 4, "cpu")
    p = torch.randn(3, 4, RECORD)
    assert torch.equal(tg.gather(p), p) and torch.equal(tg.rank_block(0), p)


@pytest.mark.parametrize("C,G,R", [(32, 1, 6), (32, 2, 8), (32, 4, 8), (32, 8, 16), (8, 2, 8),
                                   (8, 8, 8), (2, 1, 32), (2, 2, 32), (2, 4, 32), (2, 8, 32)])
def test_rig_shard_covers_the_ring_once(C, G, R):
    """The bench's streams: every (camera, ring frame) is tracked by exactly one
    rank over one pass of the ring (R frames from each stream's phase for C >= G;
    R*C/G frames of a chunk otherwise), camera blocks contiguous."""
    per_stream = R if C >= G else R * C // G
    seen = {}
    for r in range(G):
        sh = rig_shard(C, R, G, r)
        assert len(sh.cams) == max(1, C // G)
        assert list(sh.cams) == list(range(sh.cams[0], sh.cams[-1] + 1))
        for c, ph in zip(sh.cams, sh.phases):
            for t in range(per_stream):
                u = (c, (ph + t) % R)
                assert u not in seen
                seen[u] = r
    assert set(seen) == {(c, t) for c in range(C) for t in range(R)}
    al = all_streams(C, R, G)
    assert len(al.cams) == max(C, G)


def test_rig_shard_rejects():
    with pytest.raises(ValueError):
        rig_shard(2, 31, 4, 0)  # ring not divisible into 2 chunks per camera
    with pytest.raises(ValueError):
        rig_shard(3, 30, 2, 0)
