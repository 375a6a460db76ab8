"""Multi-rank paths on the one GPU of the test box (SURVEY §8(a) a7, §8(e),
§8(f) f1): ranks are separate processes sharing cuda:0 with host-side (gloo)
collectives — no kernel waits on another rank, so this is safe on one device
(the NCCL runs need a multi-GPU node; the code path above the backend is the
same).

* camera-block (C4) and frame-chunk (C2 at 4 ranks) shards of ONE seeded rig
  stream, processed with Frontend2D and the batched track-list all-gather,
  equal a single-process run over every rank's streams bit for bit;
* the rig-wide Eq. 5 keyframe decision of KeyframeTracker(group=...) over two
  ranks (half the cameras each) equals the single-process tracker's, frame by
  frame, and so do the track tables."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu

STEPS = 3


def _collect(procs, q, n):
    """n queue items, failing fast if a rank process dies first."""
    import queue
    import time
    out, t0 = [], time.time()
    while len(out) < n:
        try:
            out.append(q.get(timeout=5))
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            assert not dead, f"rank process failed: exit codes {dead}"
            assert time.time() - t0 < 600, "rank processes timed out"
    return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _small(name):
    """The config's camera count and sizes; a short ring (parity test, not bench)."""
    return synth.WORKLOADS[name]


def _run_streams(wl, cams, phases, F, R, dev, gather=None):
    """Frontend2D over the given streams for STEPS steps; returns the
    (x, y, status, ncc) records [STEPS, F*len(cams), P, 4]."""
    from paper_2506_04359_b200 import vslam2d as v2d
    from paper_2506_04359_b200.frontend import Frontend2D, RingSchedule
    cfg = v2d.FrontendConfig(W=wl.W, H=wl.H, levels=wl.levels, grid_x=wl.grid_x,
                             grid_y=wl.grid_y, k=wl.k, K_min=wl.K_min, border=wl.border,
                             win=wl.win)
    need = {(p + t) % R for p in phases for t in range(-1, STEPS * F)}
    uc = sorted(set(cams))
    st = synth.make_stream(wl, R, dev, cams=uc, only=need)
    sched = RingSchedule(st.frames, F, cams=[uc.index(c) for c in cams], phases=phases)
    fe = Frontend2D(cfg, len(cams), F, dev, wl.pitch)
    fe.prime(sched.before_first, 1)
    out = torch.zeros((STEPS, fe.B, fe.P, 4), device=dev)
    for s in range(STEPS):
        cur, prev, parity = sched.tables(s)
        rec = gather.slot(s) if gather is not None else out[s]
        fe.step(cur, prev, parity, track_list=rec)
        if gather is not None:
            gather.step_done(s)
    return out, fe


def _shard_worker(rank, world, port, name, F, R, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2506_04359_b200.shard import BatchedTrackGather, rig_shard
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = _small(name)
        sh = rig_shard(wl.cams, R, world, rank)
        dev = torch.device("cuda", 0)
        B = F * len(sh.cams)
        from paper_2506_04359_b200 import vslam2d as v2d
        P = wl.grid_x * wl.grid_y * v2d.grid_k(wl.grid_x, wl.grid_y, wl.k, wl.K_min)
        bg = BatchedTrackGather(STEPS, B, P, dev, side=torch.cuda.Stream(dev))
        _run_streams(wl, sh.cams, sh.phases, F, R, dev, gather=bg)
        bg.flush()
        torch.cuda.synchronize()
        if rank == 0:
            h = (0 // STEPS) % 2
            q.put(bg.all[h].cpu().numpy())  # [world, STEPS, B, P, 4]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world,F", [("c4", 2, 1), ("c2", 4, 2)])
def test_sharded_gather_equals_single_process(name, world, F):
    from paper_2506_04359_b200.shard import all_streams, rig_shard
    wl = _small(name)
    R = 4 * F * max(1, world // wl.cams)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, name, F, R, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = _collect(procs, q, 1)[0]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    al = all_streams(wl.cams, R, world)
    ref, fe = _run_streams(wl, al.cams, al.phases, F, R, torch.device("cuda", 0))
    torch.cuda.synchronize()
    nl = max(1, wl.cams // world)
    ref_r = ref.view(STEPS, F, world, nl, fe.P, 4).permute(2, 0, 1, 3, 4, 5).cpu().numpy()
    got_r = got.reshape(world, STEPS, F, nl, fe.P, 4)
    tracked = int((got_r[..., 2] == 0).sum())
    assert tracked > 0.5 * got_r[..., 2].size * 0.5
    assert np.array_equal(got_r, ref_r)


def _kf_worker(rank, world, port, T, n_frames, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl, C = _kf_wl()
        per = C // world
        flags, tables = _kf_run(wl, list(range(rank * per, (rank + 1) * per)), T, n_frames,
                                group=dist.group.WORLD)
        q.put((rank, flags, tables))
    finally:
        dist.destroy_process_group()


def _kf_wl():
    wl = synth.Workload("kfmr", 13, 320, 240, 4, 3, grid_x=4, grid_y=3, k=6, motion=(9.0, 6.0),
                        stereo_disparity=0.0)
    return wl, 4


def _kf_run(wl, cams, T, n_frames, group=None):
    from paper_2506_04359_b200 import vslam2d as v2d
    from paper_2506_04359_b200.frontend import KeyframeTracker
    dev = torch.device("cuda", 0)
    st = synth.make_stream(wl, n_frames, dev, cams=cams)
    cfg = v2d.FrontendConfig(W=wl.W, H=wl.H, levels=wl.levels, grid_x=wl.grid_x,
                             grid_y=wl.grid_y, k=wl.k, border=11)
    kt = KeyframeTracker(cfg, len(cams), dev, wl.pitch, T=T, min_sep=8.0, group=group)
    ptr = lambda t: v2d.ptrs_of(st.frames[:, t])
    kt.start(ptr(0))
    flags = []
    for t in range(1, n_frames):
        kt.step(ptr(t), ptr(t - 1))
        flags.append(int(kt.flag.item()))
    tr, sts, kf, ids, nid = kt.table()
    return flags, [x.cpu().numpy() for x in (tr, sts, kf, ids, nid)]


def test_keyframe_group_decision_equals_single_process():
    """Eq. 5 is rig-global ("a keyframe is still treated as a global
    event"): with half the cameras per rank and the counts all-reduced, every
    frame's decision and the final track tables equal one process's."""
    T, n_frames, world = 0.85, 10, 2
    wl, C = _kf_wl()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_kf_worker, args=(r, world, port, T, n_frames, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (f, t)) for r, f, t in _collect(procs, q, world))
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    flags1, tables1 = _kf_run(wl, list(range(C)), T, n_frames)
    print("keyframe flags per frame:", flags1)
    per = C // world
    for r in range(world):
        flags_r, tables_r = res[r]
        assert flags_r == flags1, (r, flags_r, flags1)
        for a, b in zip(tables_r, tables1):
            assert np.array_equal(a, b[r * per:(r + 1) * per])
