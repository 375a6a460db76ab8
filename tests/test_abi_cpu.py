"""CPU-side checks of the boundary: the C-ABI library builds, loads and exports
every symbol include/vslam2d.h declares; host-only entry points (layout, Eq. 1)
and argument validation behave as documented (validation returns before any
CUDA call, so these run without a GPU); the product path never touches
oracle/."""
import ctypes
import glob
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def v2d():
    from paper_2506_04359_b200 import build
    build.build()
    from paper_2506_04359_b200 import vslam2d
    return vslam2d


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "vslam2d.h")).read()
    return sorted(set(re.findall(r"\b(v2d_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(v2d):
    lib = v2d.load()
    declared = _declared_symbols()
    assert len(declared) >= 7
    for s in declared:
        assert hasattr(lib, s), s
    nm = subprocess.run(["nm", "-D", "--defined-only", v2d.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    for s in declared:
        assert re.search(rf"\bT {s}\b", nm), s


def test_library_is_sm100a(v2d):
    out = subprocess.run(["cuobjdump", "--list-elf", v2d.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_layout_matches_floor_halving(v2d):
    lay = v2d.pyramid_layout(1241, 376, 4)
    assert [lay.W[i] for i in range(4)] == [1241, 620, 310, 155]
    assert [lay.H[i] for i in range(4)] == [376, 188, 94, 47]
    for L in range(1, 4):
        assert lay.pitch[L] % 32 == 0 and lay.pitch[L] >= lay.W[L]
        assert lay.offset[L] % 32 == 0
    assert lay.offset[1] == 0
    assert lay.floats_per_image == sum(lay.pitch[L] * lay.H[L] for L in range(1, 4))


@pytest.mark.parametrize("W,H,levels", [(64, 64, 0), (64, 64, 9), (7, 64, 4), (64, 3, 3)])
def test_layout_rejects(v2d, W, H, levels):
    with pytest.raises(v2d.V2DError):
        v2d.pyramid_layout(W, H, levels)


def test_grid_k_eq1(v2d):
    assert v2d.grid_k(8, 6, 0, 300) == 7
    assert v2d.grid_k(8, 8, 0, 1000) == 16
    assert v2d.grid_k(8, 8, 0, 2000) == 32
    assert v2d.grid_k(8, 8, 0, 1500) == 24
    for bad in [(8, 8, 4, 256), (8, 8, 257, 0), (0, 8, 1, 0), (8, 8, -1, 0)]:
        with pytest.raises(v2d.V2DError):
            v2d.grid_k(*bad)


def test_validation_without_gpu(v2d):
    """Invalid arguments are rejected host-side with the documented codes."""
    L = v2d.load()
    N = None
    # build_pyramid: too many levels / bad pitch
    assert L.v2d_build_pyramid(N, 64, 0, 64, 64, 9, N, N) == -1
    assert L.v2d_build_pyramid(N, 40, 0, 33, 10, 2, N, N) == -2
    # detect: border < 3, Eq. 1 violation, nms not 0/1, grid cell < 1 px
    assert L.v2d_detect_gftt(N, 64, 0, 64, 64, 8, 8, 4, 0, 0.0, 2, 1, N, N, N, N, N, N, N, N) == -1
    assert L.v2d_detect_gftt(N, 64, 0, 64, 64, 8, 8, 4, 256, 0.0, 3, 1, N, N, N, N, N, N, N, N) == -1
    assert L.v2d_detect_gftt(N, 64, 0, 64, 64, 8, 8, 4, 0, 0.0, 3, 2, N, N, N, N, N, N, N, N) == -1
    assert L.v2d_detect_gftt(N, 64, 0, 64, 64, 65, 8, 4, 0, 0.0, 3, 1, N, N, N, N, N, N, N, N) == -1
    # klt: even window, window too large, iters < 1, bad pitch
    args = dict(eps=0.01, ncc=0.8, eig=0.01)
    f = ctypes.c_float
    assert L.v2d_track_klt(N, N, N, N, 64, 0, 64, 64, 3, N, N, N, 0, 20, 10, f(0.01), f(0.8),
                           f(0.01), N, N, N, N, N, 0, N) == -1
    assert L.v2d_track_klt(N, N, N, N, 64, 0, 64, 64, 3, N, N, N, 0, 31, 10, f(0.01), f(0.8),
                           f(0.01), N, N, N, N, N, 0, N) == -1
    assert L.v2d_track_klt(N, N, N, N, 64, 0, 64, 64, 3, N, N, N, 0, 21, 0, f(0.01), f(0.8),
                           f(0.01), N, N, N, N, N, 0, N) == -1
    assert L.v2d_track_klt(N, N, N, N, 72, 0, 70, 64, 3, N, N, N, 0, 21, 10, f(0.01), f(0.8),
                           f(0.01), N, N, N, N, N, 0, N) == -2
    # min_eig <= 0 or NaN (reading #27), B*P beyond the grid limit, unaligned track_list
    for me in (0.0, -1.0, float("nan")):
        assert L.v2d_track_klt(N, N, N, N, 64, 0, 64, 64, 3, N, N, N, 0, 21, 10, f(0.01),
                               f(0.8), f(me), N, N, N, N, N, 0, N) == -1
    assert L.v2d_track_klt(N, N, N, N, 64, 65536, 64, 64, 3, N, N, N, 65536, 21, 10, f(0.01),
                           f(0.8), f(0.01), N, N, N, N, N, 0, N) == -1
    assert L.v2d_track_klt(N, N, N, N, 64, 0, 64, 64, 3, N, N, N, 0, 21, 10, f(0.01), f(0.8),
                           f(0.01), N, N, N, N, ctypes.c_void_p(8), 0, N) == -2
    assert L.v2d_extract_patches(N, N, 64, 65536, 64, 64, 3, N, 65536, 9, N, N) == -1
    # empty batches are valid no-ops (no CUDA call is made for B == 0)
    assert L.v2d_build_pyramid(N, 64, 0, 64, 64, 3, N, N) == 0
    assert L.v2d_strerror(-2).decode().startswith("pitch")
    assert L.v2d_version() == 201
    del args


def test_product_path_never_touches_oracle():
    pkg = os.path.join(ROOT, "paper_2506_04359_b200")
    for path in glob.glob(os.path.join(pkg, "**", "*.*"), recursive=True):
        if path.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
            txt = open(path).read()
            assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), path
            assert "v2dref" not in txt, path
    ldd = subprocess.run(["ldd", os.path.join(pkg, "libvslam2d.so")], capture_output=True,
                         text=True).stdout
    assert "v2dref" not in ldd


def test_oracle_and_product_share_no_sources():
    ora = {os.path.basename(p) for p in glob.glob(os.path.join(ROOT, "oracle", "*"))}
    prod = {os.path.basename(p) for p in glob.glob(os.path.join(ROOT, "paper_2506_04359_b200",
                                                                "**", "*"), recursive=True)}
    assert not ({n for n in ora if not n.startswith("__")} & prod)


def test_binding_requires_cuda_tensors(v2d):
    import torch
    with pytest.raises((v2d.V2DError, RuntimeError, AssertionError)):
        v2d.build_pyramid(torch.zeros((1, 16, 16), dtype=torch.uint8), 16, 2)


def test_keyframe_calls_validate_without_gpu(v2d):
    L = v2d.load()
    N = None
    f = ctypes.c_float
    assert L.v2d_suppress_mask(N, N, 1, 4, f(5.0), 64, 64, N, 64, N, N) == -1   # null mask ptrs
    assert L.v2d_suppress_mask(N, N, 0, 0, f(5.0), 64, 64, N, 40, N, N) == -2   # pitch % 16
    assert L.v2d_keyframe_decide(N, 0, f(0.7), N, N, N) == -1                   # null flag
    assert L.v2d_refill_tracks(N, N, 64, 32, 4, N, 0, 0, N, N, N, N, N, N) == -1  # > 1024 cells
    assert L.v2d_extract_patches(N, N, 64, 0, 64, 64, 2, N, 0, 8, N, N) == -1   # even patch
    assert L.v2d_keyframe_decide_graph(N, 0, f(0.7), N, N, N, 0, N) == -1      # null flag
    assert L.v2d_keyframe_decide_graph(N, 0, f(-1.0), N, N, N, 0, N) == -1     # T < 0
    assert L.v2d_ring_tables(N, 0, 2, N, N, N, N) == -1                         # R < 1
    assert L.v2d_ring_tables(N, 4, 2, N, N, N, N) == -1                         # null table
