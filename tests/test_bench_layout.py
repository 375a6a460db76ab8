"""bench.py's per-rank work layout (CPU): every config and GPU count gives a ring
that is a multiple of 2F (pyramid double buffer) and of the frame-chunk count,
holds >= 2.5x L2 of frames per rank (each step reads new frames from HBM),
32 camera-frames per rank and step (weak scaling), >= 16 frames per all-gather,
and both bench arms report the same config object."""
import pytest

import bench
import synth


@pytest.mark.parametrize("name", sorted(synth.WORKLOADS))
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_layout_invariants(name, world):
    wl = synth.WORKLOADS[name]
    if wl.cams < world and world % wl.cams:
        pytest.skip("not a supported partition")
    if wl.cams >= world and wl.cams % world:
        pytest.skip("not a supported partition")
    lay = bench.bench_layout(wl, world)
    per_cam = max(1, world // wl.cams)
    assert lay["R"] % (2 * lay["F"]) == 0 and lay["R"] % per_cam == 0
    assert lay["streams"] * lay["R"] * wl.H * wl.pitch >= 2.5 * bench.L2_BYTES
    assert lay["B"] == lay["F"] * lay["streams"] and lay["B"] >= 32
    assert lay["gather_steps"] * lay["F"] >= 16
    cfg = bench.workload_config(wl, lay, world)
    assert cfg == bench.workload_config(wl, bench.bench_layout(wl, world), world)
    assert cfg["camera_frames_per_step_per_gpu"] == lay["B"]


def test_default_is_the_north_star_rig():
    assert bench.DEFAULT_CONFIG == "c5"
    wl = synth.WORKLOADS["c5"]
    assert (wl.cams, wl.W, wl.H, wl.levels) == (32, 1920, 1200, 5)
