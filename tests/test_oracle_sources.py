"""Pins for the oracle's feature SOURCE switch: LBP codes computed on the u16
depth plane (Table 1's "Depth Image" row; S:559 `source: depth`) and the fused
grey||depth descriptor (the title's "fusion of RGB and depth image").  Run without a
GPU.  The depth source is pinned to the grey source (already pinned to Fig. 7 and the closed
forms in test_oracle.py) through monotone maps of the samples, and by brute force on tiny
u16 inputs that use the full 16-bit range."""
import numpy as np
import pytest

import oracle
import synthgen

# Fig. 7 sampling points (row, col offset) -> weight; restated for the brute force below
_FIG7 = [((-1, -1), 1), ((-1, 0), 2), ((-1, 1), 4), ((0, 1), 8), ((1, 1), 16), ((1, 0), 32),
         ((1, -1), 64), ((0, -1), 128)]


def _codes(plane):
    """Eq. 2 with S(x) = [x >= 0] at every interior pixel of a 2-D array (any int dtype)."""
    p = plane.astype(np.int64)
    H, W = p.shape
    c = p[1:-1, 1:-1]
    code = np.zeros_like(c)
    for (dy, dx), w in _FIG7:
        code += (p[1 + dy:H - 1 + dy, 1 + dx:W - 1 + dx] >= c) * w
    return code


def test_depth_source_equals_grey_source_under_increasing_map():
    """Eq. 2 depends only on the ORDER of the samples: if depth = phi(grey) with phi
    strictly increasing, the depth-source descriptor equals the grey-source one (same mask)."""
    grey, _ = synthgen.face_crops(3, 48, 40, seed=11)
    depth = (650 + 3 * grey.astype(np.uint16)).astype(np.uint16)  # 650..1415 mm
    rois = synthgen.full_rois(3, 48, 40)
    for bins in (59, 256):
        g = oracle.lbp_extract(grey, depth, rois, 600, 1400, 5, 4, bins)
        d = oracle.lbp_extract(grey, depth, rois, 600, 1400, 5, 4, bins, source=oracle.SRC_DEPTH)
        assert g.sum() > 0 and np.array_equal(g, d)


def test_depth_source_complement_under_decreasing_map():
    """For a strictly DECREASING map and windows without ties every bit flips: code' = 255 -
    code (256 bins).  Pixels with a tie in the window are excluded by construction: the
    grey plane is a permutation of distinct values."""
    rng = np.random.default_rng(3)
    H, W = 12, 14
    grey = rng.permutation(H * W).astype(np.uint8).reshape(1, H, W)  # 168 distinct values
    depth = (30000 - 7 * grey.astype(np.uint16)).astype(np.uint16)
    rois = [[0, 0, 0, W, H]]
    g = oracle.lbp_extract(grey, None, rois, 0, 0, 1, 1, 256)[0]
    d = oracle.lbp_extract(grey, depth, rois, 1, 65535, 1, 1, 256, source=oracle.SRC_DEPTH)[0]
    assert np.array_equal(d, g[::-1])  # count of code c moves to 255 - c


def test_depth_source_brute_force_full_u16_range():
    """Tiny crops, every grid, samples spanning 0..65535 (holes, far values, ties)."""
    rng = np.random.default_rng(5)
    vals = np.array([0, 1, 255, 256, 1000, 1001, 2047, 2048, 40000, 65534, 65535], np.uint16)
    for H in range(3, 7):
        for W in range(3, 7):
            depth = vals[rng.integers(0, len(vals), (1, H, W))]
            grey = np.zeros((1, H, W), np.uint8)
            codes = _codes(depth[0])
            dd = depth[0, 1:-1, 1:-1].astype(np.int64)
            valid = (dd != 0) & (dd >= 1) & (dd <= 65535)
            for kx in range(1, W - 1):
                for ky in range(1, H - 1):
                    desc = oracle.lbp_extract(grey, depth, [[0, 0, 0, W, H]], 1, 65535, kx, ky,
                                              256, source=oracle.SRC_DEPTH)
                    expect = np.zeros((ky, kx, 256), np.int64)
                    for i in range(H - 2):
                        for j in range(W - 2):
                            if valid[i, j]:
                                expect[_cell(i, H - 2, ky), _cell(j, W - 2, kx), codes[i, j]] += 1
                    assert np.array_equal(desc.reshape(ky, kx, 256), expect)


def _cell(i, n, k):
    """Block b spans [floor(b*n/k), floor((b+1)*n/k)): the b containing i."""
    for b in range(k):
        if (b * n) // k <= i < ((b + 1) * n) // k:
            return b
    raise AssertionError


def test_fused_is_grey_then_depth_block():
    grey, depth = synthgen.face_crops(4, 64, 64, seed=21)
    rois = synthgen.full_rois(4, 64, 64)
    g = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 59)
    d = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 59, source=oracle.SRC_DEPTH)
    f, st = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 59, source=oracle.SRC_FUSED,
                               return_status=True)
    assert f.shape == (4, 2 * 8 * 8 * 59) and (st == 0).all()
    assert np.array_equal(f[:, :g.shape[1]], g) and np.array_equal(f[:, g.shape[1]:], d)
    # both blocks count the same valid pixels (the mask gates the centre in both)
    assert np.array_equal(g.reshape(4, 64, 59).sum(2), d.reshape(4, 64, 59).sum(2))


def test_depth_source_constant_plane_and_errors():
    """A flat depth plane inside the window: every valid pixel has code 255 (all ties,
    S(0) = 1); errors: depth source needs a depth plane; bad source value."""
    grey = np.zeros((1, 20, 20), np.uint8)
    depth = np.full((1, 20, 20), 900, np.uint16)
    d = oracle.lbp_extract(grey, depth, [[0, 0, 0, 20, 20]], 600, 1400, 2, 2, 59,
                           source=oracle.SRC_DEPTH).reshape(4, 59)
    assert (d[:, 57] == 81).all() and d.sum() == 324
    with pytest.raises(ValueError):
        oracle.lbp_extract(grey, None, [[0, 0, 0, 20, 20]], 0, 0, 2, 2, 59,
                           source=oracle.SRC_DEPTH)
    with pytest.raises(ValueError):
        oracle.lbp_extract(grey, depth, [[0, 0, 0, 20, 20]], 0, 0, 2, 2, 59, source=3)
