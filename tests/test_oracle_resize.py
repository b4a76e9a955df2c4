"""Pins for the oracle's ROI resize ("resized to 200x200 pixels"):
grey bilinear with half-pixel centres rounded half up, depth nearest neighbour with
half-pixel centres and ties toward the smaller index, and the resized-ROI descriptor.
The C oracle works in exact integers; the brute force below follows the textbook formula in
exact rationals (fractions.Fraction), a different derivation."""
from fractions import Fraction as F

import numpy as np
import pytest

import oracle
import synthgen


def _bilinear_ref(img, out_h, out_w):
    h, w = img.shape
    out = np.zeros((out_h, out_w), np.int64)
    for oy in range(out_h):
        sy = max(F(2 * oy + 1, 2) * F(h, out_h) - F(1, 2), F(0))
        y0 = min(int(sy), h - 1)  # floor (sy >= 0)
        fy = sy - y0 if int(sy) <= h - 1 else F(0)
        y1 = min(y0 + 1, h - 1)
        for ox in range(out_w):
            sx = max(F(2 * ox + 1, 2) * F(w, out_w) - F(1, 2), F(0))
            x0 = min(int(sx), w - 1)
            fx = sx - x0 if int(sx) <= w - 1 else F(0)
            x1 = min(x0 + 1, w - 1)
            v = ((1 - fx) * (1 - fy) * int(img[y0, x0]) + fx * (1 - fy) * int(img[y0, x1]) +
                 (1 - fx) * fy * int(img[y1, x0]) + fx * fy * int(img[y1, x1]))
            out[oy, ox] = int(v + F(1, 2)) if v + F(1, 2) >= 0 else -1  # floor, v >= 0
    return out


def _nearest_ref(img, out_h, out_w):
    """Nearest source index to s = (o + 1/2) * n / m - 1/2; ties -> the smaller index."""
    h, w = img.shape

    def pick(o, n, m):
        s = F(2 * o + 1, 2) * F(n, m) - F(1, 2)
        best = None
        for i in range(n):
            dist = abs(F(i) - s)
            if best is None or dist < best[0]:
                best = (dist, i)
        return best[1]
    ys = [pick(oy, h, out_h) for oy in range(out_h)]
    xs = [pick(ox, w, out_w) for ox in range(out_w)]
    return img[np.ix_(ys, xs)]


def test_spec_examples():
    """identity at the same size; 1x1 value 7 -> 3x3 of 7; 2x1 [0,100] -> 4x1."""
    rng = np.random.default_rng(1)
    g = rng.integers(0, 256, (7, 9)).astype(np.uint8)
    d = rng.integers(0, 65536, (7, 9)).astype(np.uint16)
    assert np.array_equal(oracle.resize_grey(g, 7, 9), g)
    assert np.array_equal(oracle.resize_depth(d, 7, 9), d)
    assert (oracle.resize_grey(np.full((1, 1), 7, np.uint8), 3, 3) == 7).all()
    assert oracle.resize_grey(np.array([[0, 100]], np.uint8), 1, 4).tolist() == [[0, 25, 75, 100]]


def test_rounding_ties_and_nearest_ties():
    """Round half up: [0, 1] -> 1 px samples 0.5 -> 1.  Nearest ties go to the smaller index:
    [10, 20] -> 1 px = 10; 4 -> 2 px picks indices 0 and 2."""
    assert oracle.resize_grey(np.array([[0, 1]], np.uint8), 1, 1).tolist() == [[1]]
    assert oracle.resize_depth(np.array([[10, 20]], np.uint16), 1, 1).tolist() == [[10]]
    assert oracle.resize_depth(np.arange(4, dtype=np.uint16)[None], 1, 2).tolist() == [[0, 2]]


@pytest.mark.parametrize("h,w,oh,ow", [(5, 7, 11, 3), (9, 4, 4, 9), (3, 3, 8, 8), (13, 6, 5, 5),
                                       (2, 11, 7, 17), (6, 6, 6, 13), (1, 5, 3, 2)])
def test_brute_force_exact_rationals(h, w, oh, ow):
    rng = np.random.default_rng(h * 100 + w * 10 + oh)
    g = rng.integers(0, 256, (h, w)).astype(np.uint8)
    d = rng.integers(0, 65536, (h, w)).astype(np.uint16)
    assert np.array_equal(oracle.resize_grey(g, oh, ow).astype(np.int64), _bilinear_ref(g, oh, ow))
    assert np.array_equal(oracle.resize_depth(d, oh, ow), _nearest_ref(d, oh, ow))


def test_invariants():
    """Constant -> constant; depth output values come from the input (never blended);
    grey resize commutes with a horizontal flip (the half-pixel mapping is symmetric and the
    interpolated value is the same rational, so it rounds the same way); a monotone ramp
    stays monotone."""
    assert (oracle.resize_grey(np.full((5, 8), 200, np.uint8), 13, 3) == 200).all()
    assert (oracle.resize_depth(np.full((5, 8), 777, np.uint16), 2, 19) == 777).all()
    rng = np.random.default_rng(7)
    d = rng.integers(0, 5000, (23, 31)).astype(np.uint16)
    d[rng.random(d.shape) < 0.2] = 0
    r = oracle.resize_depth(d, 200, 200)
    assert set(np.unique(r)) <= set(np.unique(d))
    g = rng.integers(0, 256, (37, 29)).astype(np.uint8)
    for oh, ow in ((200, 200), (16, 50), (61, 7)):
        assert np.array_equal(oracle.resize_grey(g[:, ::-1], oh, ow),
                              oracle.resize_grey(g, oh, ow)[:, ::-1])
    ramp = np.tile(np.arange(0, 250, 10, dtype=np.uint8), (3, 1))
    out = oracle.resize_grey(ramp, 3, 97)
    assert (np.diff(out.astype(int), axis=1) >= 0).all()


def test_resized_descriptor_identity_and_clamp():
    """size == ROI side on an in-bounds square ROI is the plain descriptor; a clamped ROI is
    resized from its intersection; an empty ROI is E_ROI with a zero row."""
    grey, depth = synthgen.face_crops(2, 240, 320, seed=3)
    rois = [[0, 40, 30, 128, 128], [1, 100, 50, 96, 96]]
    for src in (0, 1, 2):
        a = oracle.lbp_extract_resized(grey, depth, rois[:1], 128, 600, 1400, 8, 8, 59,
                                       source=src)
        b = oracle.lbp_extract(grey, depth, rois[:1], 600, 1400, 8, 8, 59, source=src)
        assert np.array_equal(a, b)
    # clamped ROI: resize of the manual crop of the intersection
    r, st = oracle.lbp_extract_resized(grey, depth, [[1, 280, -10, 100, 80]], 64, 600, 1400, 4,
                                       4, 256, return_status=True)
    g = oracle.resize_grey(grey[1, 0:70, 280:320], 64, 64)
    d = oracle.resize_depth(depth[1, 0:70, 280:320], 64, 64)
    ref = oracle.lbp_extract(g, d, [[0, 0, 0, 64, 64]], 600, 1400, 4, 4, 256)
    assert st.tolist() == [0] and np.array_equal(r, ref)
    r, st = oracle.lbp_extract_resized(grey, depth, [[0, 400, 0, 10, 10], [0, 5, 5, 1, 1]], 32,
                                       600, 1400, 2, 2, 59, return_status=True)
    assert st.tolist() == [-2, 0] and r[0].sum() == 0
    # a 1x1 crop resized to 32x32 is a constant grey image: every valid pixel has code 255
    assert r[1].reshape(4, 59)[:, :57].sum() == 0


def test_resized_argument_errors():
    g = np.zeros((1, 8, 8), np.uint8)
    with pytest.raises(ValueError):
        oracle.lbp_extract_resized(g, None, [[0, 0, 0, 8, 8]], 2, 0, 0, 1, 1, 59)  # size < 3
    with pytest.raises(ValueError):
        oracle.lbp_extract_resized(g, None, [[0, 0, 0, 8, 8]], 8, 0, 0, 1, 1, 59, source=1)
