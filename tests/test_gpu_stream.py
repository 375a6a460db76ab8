"""The public host-streaming API (frontend.HostStream: pipelined H2D / kernels /
D2H on two streams) returns exactly what the device-resident frontend computes
for the same frames, step by step (bit-identical keypoints, positions and
statuses): the overlap changes timing only."""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def test_host_stream_matches_device_frontend():
    from paper_2506_04359_b200 import vslam2d as v2d
    from paper_2506_04359_b200.frontend import Frontend2D, HostStream
    wl = synth.WORKLOADS["c2"]
    C, F, steps = wl.cams, 2, 6
    st = synth.make_stream(wl, F * (steps + 1), "cuda")
    frames = st.frames  # [C, R, H, pitch]
    B = F * C

    def batch(s):  # batch of step s (s = -1: the priming batch), order f*C + c
        return torch.stack([frames[c, (s + 1) * F + f] for f in range(F) for c in range(C)])

    cfg = v2d.FrontendConfig(W=wl.W, H=wl.H, levels=wl.levels, grid_x=wl.grid_x,
                             grid_y=wl.grid_y, k=wl.k, K_min=wl.K_min, border=wl.border,
                             win=wl.win, iters=wl.iters, eps=wl.eps, ncc_min=wl.ncc_min,
                             min_eig=wl.min_eig)
    # reference: device-resident frames, one stream
    fe_ref = Frontend2D(cfg, C, F, "cuda", wl.pitch)
    dev_batches = [batch(s).contiguous() for s in range(-1, steps)]
    ptrs = [v2d.ptrs_of(b) for b in dev_batches]
    fe_ref.prime(ptrs[0][-C:], 1)
    ref = []
    for s in range(steps):
        cur, prv = ptrs[s + 1], torch.empty_like(ptrs[s + 1])
        prv[C:] = cur[:-C]
        prv[:C] = ptrs[s][-C:]
        fe_ref.step(cur, prv, s % 2)
        ref.append((fe_ref.kp_xy[1:].clone(), fe_ref.pos.clone(), fe_ref.status.clone()))
    torch.cuda.synchronize()
    # pipelined host stream
    host = [b.cpu().pin_memory() for b in dev_batches]
    fe = Frontend2D(cfg, C, F, "cuda", wl.pitch)
    hs = HostStream(fe)
    hs.start(host[0])
    hs.upload(0, host[1])
    for s in range(steps):
        if s + 1 < steps:
            hs.upload(s + 1, host[s + 2])
        hs.compute(s)
        hs.download(s)
        kp, pos, status = hs.results(s)
        assert torch.equal(kp, ref[s][0].cpu()), s
        assert torch.equal(pos, ref[s][1].cpu()), s
        assert torch.equal(status, ref[s][2].cpu()), s
    hs.finish()
    torch.cuda.synchronize()
    assert B == hs.h2d_bytes_per_step // (wl.H * wl.pitch)


def test_keyframe_tracker_graph_replay_matches_eager():
    """f1 replayed as CUDA graphs (device-side frame tables) == eager steps."""
    from paper_2506_04359_b200 import vslam2d as v2d
    from paper_2506_04359_b200.frontend import KeyframeTracker
    wl = synth.WORKLOADS["c2"]
    C, n = wl.cams, 12
    st = synth.make_stream(wl, n, "cuda")
    img = st.frames.stride(1) * st.frames.element_size()
    cam = st.frames.stride(0) * st.frames.element_size()
    t = torch.arange(n, device="cuda", dtype=torch.int64)[:, None]
    c = torch.arange(C, device="cuda", dtype=torch.int64)[None, :]
    table = (st.frames.data_ptr() + c * cam + t * img).contiguous()  # [n, C]
    cfg = v2d.FrontendConfig(W=wl.W, H=wl.H, levels=wl.levels, grid_x=wl.grid_x,
                             grid_y=wl.grid_y, k=wl.k, K_min=wl.K_min, border=wl.border,
                             win=wl.win, iters=wl.iters, eps=wl.eps, ncc_min=wl.ncc_min,
                             min_eig=wl.min_eig)
    eager = KeyframeTracker(cfg, C, "cuda", wl.pitch, T=0.7)
    graph = KeyframeTracker(cfg, C, "cuda", wl.pitch, T=0.7)
    for kt in (eager, graph):
        kt.start(table[0])
        kt.step(table[1], table[0])
    for f in range(2, n):
        eager.step(table[f], table[f - 1])
    graph.capture(table, 2)
    # the keyframe branch is a conditional (IF) graph node set by the decide kernel
    assert graph.graph_kind == "conditional", getattr(graph, "graph_fallback_reason", "")
    for f in range(2, n):
        graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager.table(), graph.table()):
        assert torch.equal(a, b)


def test_keyframe_tracker_torch_graph_fallback_matches_eager():
    """The torch.cuda.graph capture (no conditional node: the branch's kernels exit on
    the device flag) gives the same tables as eager steps."""
    from paper_2506_04359_b200 import vslam2d as v2d
    from paper_2506_04359_b200.frontend import KeyframeTracker
    wl = synth.WORKLOADS["c2"]
    C, n = wl.cams, 10
    st = synth.make_stream(wl, n, "cuda")
    img = st.frames.stride(1) * st.frames.element_size()
    cam = st.frames.stride(0) * st.frames.element_size()
    t = torch.arange(n, device="cuda", dtype=torch.int64)[:, None]
    c = torch.arange(C, device="cuda", dtype=torch.int64)[None, :]
    table = (st.frames.data_ptr() + c * cam + t * img).contiguous()
    cfg = v2d.FrontendConfig(W=wl.W, H=wl.H, levels=wl.levels, grid_x=wl.grid_x,
                             grid_y=wl.grid_y, k=wl.k, K_min=wl.K_min, border=wl.border,
                             win=wl.win, iters=wl.iters, eps=wl.eps, ncc_min=wl.ncc_min,
                             min_eig=wl.min_eig)
    eager = KeyframeTracker(cfg, C, "cuda", wl.pitch, T=0.9)
    graph = KeyframeTracker(cfg, C, "cuda", wl.pitch, T=0.9)
    for kt in (eager, graph):
        kt.start(table[0])
        kt.step(table[1], table[0])
    for f in range(2, n):
        eager.step(table[f], table[f - 1])
    graph.capture(table, 2, conditional=False)
    assert graph.graph_kind == "torch"
    for f in range(2, n):
        graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager.table(), graph.table()):
        assert torch.equal(a, b)


@pytest.mark.parametrize("name,F", [("c2", 1), ("c2", 4), ("c4", 1)])
def test_overlap_streams_match_serial(name, F):
    """Frontend2D(overlap=True) — the first frame's KLT launch on a second stream,
    concurrent with detection — gives bit-identical keypoints, positions,
    statuses, NCC and track-list records to the serial step, over several steps
    (so the cross-stream ordering of the pyramid double buffer and the keypoint
    carry is right)."""
    from paper_2506_04359_b200 import vslam2d as v2d
    from paper_2506_04359_b200.frontend import Frontend2D, RingSchedule
    wl = synth.WORKLOADS[name]
    C, steps = wl.cams, 4
    st = synth.make_stream(wl, 2 * F * steps, "cuda")
    cfg = v2d.FrontendConfig(W=wl.W, H=wl.H, levels=wl.levels, grid_x=wl.grid_x,
                             grid_y=wl.grid_y, k=wl.k, K_min=wl.K_min, border=wl.border,
                             win=wl.win)
    outs = []
    for overlap in (False, True):
        fe = Frontend2D(cfg, C, F, "cuda", wl.pitch, overlap=overlap)
        sched = RingSchedule(st.frames, F)
        fe.prime(sched.before_first, 1)
        rec = torch.zeros((steps, fe.B, fe.P, 4), device="cuda")
        res = []
        for s in range(steps):
            cur, prev, parity = sched.tables(s)
            fe.step(cur, prev, parity, track_list=rec[s])
            res.append([x.clone() for x in (fe.kp_xy, fe.pos, fe.status, fe.ncc)])
        torch.cuda.synchronize()
        outs.append((res, rec))
    for s in range(steps):
        for a, b in zip(outs[0][0][s], outs[1][0][s]):
            assert torch.equal(a, b), s
    assert torch.equal(outs[0][1], outs[1][1])
    assert int((outs[0][1][..., 2] == 0).sum()) > 0


def test_ring_tables_and_decide_graph_counter():
    """v2d_ring_tables: rows t and t-1 (mod R, t = 0 wraps to row R-1) of the pointer
    table, counter advanced; v2d_keyframe_decide_graph outside a graph (handle 0): the
    Eq. 5 flag of v2d_keyframe_decide and kf_count += flag."""
    from paper_2506_04359_b200 import vslam2d as v2d
    R, C = 5, 3
    table = torch.arange(R * C, dtype=torch.int64, device="cuda").view(R, C) * 16 + 4096
    counter = torch.zeros((1,), dtype=torch.int64, device="cuda")
    cur = torch.empty((C,), dtype=torch.int64, device="cuda")
    prev = torch.empty_like(cur)
    for t in range(2 * R + 1):
        v2d.ring_tables(table, counter, cur, prev)
        torch.cuda.synchronize()
        assert torch.equal(cur, table[t % R]) and torch.equal(prev, table[(t - 1) % R]), t
        assert int(counter.item()) == t + 1
    counts = torch.tensor([[10, 6], [10, 8]], dtype=torch.int32, device="cuda")  # 14/20 = 0.7
    flag = torch.zeros((1,), dtype=torch.int32, device="cuda")
    ref = torch.zeros_like(flag)
    kf = torch.zeros((), dtype=torch.int64, device="cuda")
    for T, want in ((0.71, 1), (0.7, 0), (0.69, 0), (1.0, 1)):
        v2d.keyframe_decide_graph(counts, T, flag, None, kf)
        v2d.keyframe_decide(counts, T, ref)
        torch.cuda.synchronize()
        assert int(flag.item()) == want == int(ref.item()), T
    assert int(kf.item()) == 2


def test_survival_decide_matches_survival_then_decide():
    """v2d_survival_decide (one launch, last-block decision) == v2d_track_survival +
    v2d_keyframe_decide on random tables, repeatedly (the done counter returns to 0)."""
    from paper_2506_04359_b200 import vslam2d as v2d
    g = torch.Generator(device="cpu").manual_seed(3)
    done = torch.zeros((1,), dtype=torch.int32, device="cuda")
    kf = torch.zeros((), dtype=torch.int64, device="cuda")
    n_kf = 0
    for it in range(12):
        B, P = [(1, 5), (7, 300), (32, 2048), (3, 1)][it % 4]
        status = torch.randint(0, 5, (B, P), generator=g, dtype=torch.uint8).cuda()
        member = (torch.rand((B, P), generator=g) < 0.6).to(torch.uint8).cuda()
        if it == 5:
            member.zero_()  # bootstrap: no keyframe members -> keyframe
        T = [0.3, 0.7, 0.9, 1.01][it % 4]
        c1 = torch.zeros((B, 2), dtype=torch.int32, device="cuda")
        c2 = torch.zeros_like(c1)
        f1 = torch.zeros((1,), dtype=torch.int32, device="cuda")
        f2 = torch.zeros_like(f1)
        t1 = torch.zeros((2,), dtype=torch.int64, device="cuda")
        t2 = torch.zeros_like(t1)
        v2d.survival_decide(status, member, c1, T, f1, done, t1, kf)
        v2d.track_survival(status, member, c2)
        v2d.keyframe_decide(c2, T, f2, t2)
        torch.cuda.synchronize()
        assert torch.equal(c1, c2) and torch.equal(f1, f2) and torch.equal(t1, t2), it
        assert int(done.item()) == 0
        n_kf += int(f2.item())
    assert int(kf.item()) == n_kf
