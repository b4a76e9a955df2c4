"""GPU parity of the three depth-window tests of the lane-private TMA kernel (lbp_hist_lane59.cuh
WINM 0: integer compare; 1: fp16 >= dmin and <= dmax on the raw words, dmax <= 0x7BFE; 2:
|d - mid| <= half, dmax < 2048 and dmin + dmax even) against the oracle, bit-exact, with depth
values at and around every boundary of every window and bit patterns that are +inf, NaN or
negative as fp16 (>= 0x7C00).  Grey and depth codes, crop stacks and frames (FRAME variant)."""
import numpy as np
import pytest
import torch

import oracle
import synthgen

pytestmark = pytest.mark.gpu
DEV = "cuda"

WINDOWS = [(600, 1400),      # mode 2 (the default window)
           (601, 1400),      # mode 1: odd sum
           (600, 3000),      # mode 1: dmax >= 2048
           (1, 2047),        # mode 2: widest centred window
           (2, 2046), (1000, 1000), (0, 2046),  # mode 2 (half 0), mode 1 (dmin 0 -> 1, odd sum)
           (0x7BFE, 0x7BFE), (1, 0x7BFE),       # mode 1 at the top of its range
           (5, 40000), (0x7BFF, 0xFFFF)]        # mode 0 (integer)


@pytest.fixture(scope="module")
def lb():
    import paper_1504_01883_b200 as lb
    lb.lbpfused.lib()
    return lb


def _edge_depth(n, H, W, seed):
    """depth planes mixing a smooth face-like surface with boundary values of every window"""
    rng = np.random.default_rng(seed)
    specials = set()
    for lo, hi in WINDOWS:
        for v in (lo - 1, lo, lo + 1, hi - 1, hi, hi + 1, (lo + hi) // 2, (lo + hi + 1) // 2):
            if 0 <= v <= 0xFFFF:
                specials.add(v)
    specials |= {0, 1, 2047, 2048, 2049, 4095, 4096, 0x7BFE, 0x7BFF, 0x7C00, 0x7C01, 0x7FFF,
                 0x8000, 0x8001, 0xFBFF, 0xFC00, 0xFFFF}
    specials = np.array(sorted(specials), np.uint16)
    _, depth = synthgen.face_crops(n, H, W, seed=seed)
    pick = rng.random((n, H, W))
    depth = np.where(pick < 0.35, specials[rng.integers(0, len(specials), (n, H, W))], depth)
    depth = np.where((pick >= 0.35) & (pick < 0.45), rng.integers(0, 65536, (n, H, W)), depth)
    return depth.astype(np.uint16)


def _check(lb, grey, depth, rois, lo, hi, source):
    g = torch.from_numpy(np.ascontiguousarray(grey)).to(DEV)
    d = torch.from_numpy(np.ascontiguousarray(depth).view(np.int16)).to(DEV).view(torch.uint16)
    r = torch.from_numpy(rois).to(DEV)
    out = lb.lbp_extract_source(g, d, r, lo, hi, 8, 8, 59, source)
    torch.cuda.synchronize()
    got = out.cpu().view(torch.int16).numpy().view(np.uint16)
    ref = oracle.lbp_extract(grey, depth, rois, lo, hi, 8, 8, 59, source=source)
    bad = np.nonzero((got != ref).any(1))[0]
    assert bad.size == 0, f"window [{lo}, {hi}] source {source}: {bad.size} rows differ"


@pytest.mark.parametrize("lo,hi", WINDOWS)
def test_crop_stack_windows(lb, lo, hi):
    grey, _ = synthgen.face_crops(160, 128, 128, seed=61)
    depth = _edge_depth(160, 128, 128, 62)
    rois = synthgen.full_rois(160, 128, 128)
    _check(lb, grey, depth, rois, lo, hi, 0)
    if hi <= 0x7BFE:  # the depth-source TMA kernel's range (others take the generic kernel)
        _check(lb, grey, depth, rois, lo, hi, 1)


@pytest.mark.parametrize("lo,hi", [(600, 1400), (601, 1400), (1, 0x7BFE), (5, 40000)])
def test_frame_windows(lb, lo, hi):
    grey, _ = synthgen.face_crops(6, 240, 320, seed=63)
    depth = _edge_depth(6, 240, 320, 64)
    rng = np.random.default_rng(65)
    rois = np.array([[f, int(rng.integers(0, 193)), int(rng.integers(0, 113)), 128, 128]
                     for f in range(6) for _ in range(26)], np.int32)
    for source in (0, 1):
        _check(lb, grey, depth, rois, lo, hi, source)
