"""Pins for the CPU oracle (oracle/lbp_oracle.c) -- run without a GPU.

Each test pins the oracle to something other than itself: a value the paper
prints (Fig. 7, tests/golden/fig7_lbp.txt), a closed form, an invariant, a
metamorphic relation, brute force on tiny inputs, or exact arithmetic within
the fp32 rounding bound.  Citations: P:L = PAPER.md line, S:L = SPEC.md line.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synthgen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "fig7_lbp.txt")


def _golden_fig7():
    rows = [ln.split() for ln in open(GOLDEN) if ln.strip() and not ln.startswith("#")]
    window = np.array(rows[0:3], dtype=np.int64)
    thresholded = np.array(rows[3:6], dtype=np.int64)
    weights = np.array(rows[6:9], dtype=np.int64)
    assert rows[9][0] == "code"
    return window, thresholded, weights, int(rows[9][1])


def rotl8(c, k):
    c = np.asarray(c, dtype=np.int64)
    return ((c << k) | (c >> (8 - k))) & 0xFF


# --------------------------------------------------------------------------- Eq. 2 / Fig. 7

def test_fig7_worked_example():
    """window [[6,5,2],[7,6,1],[9,8,7]] -> LBP 241."""
    window, thresholded, weights, code = _golden_fig7()
    assert oracle.lbp_code_window(window) == code == 241
    # the printed thresholded pattern, weighted by the printed weights, is the code
    assert int(((thresholded == 1) * weights).sum()) == code


def test_fig7_weight_layout_each_position():
    """Each Fig. 7 weight individually: only neighbour p >= centre -> code = weight_p."""
    _, _, weights, _ = _golden_fig7()
    for r in range(3):
        for c in range(3):
            if (r, c) == (1, 1):
                continue
            win = np.zeros((3, 3), np.int64)
            win[1, 1] = 5
            win[r, c] = 9
            assert oracle.lbp_code_window(win) == weights[r, c]
            win[r, c] = 5  # equal -> S(0) = 1 (Fig. 7's 6-vs-6 cell)
            assert oracle.lbp_code_window(win) == weights[r, c]


def test_special_windows():
    """constant -> 255; strict max centre -> 0 (incl. u16 65535); strict min -> 255."""
    assert oracle.lbp_code_window(np.full(9, 77)) == 255
    w = np.arange(9)
    w[4] = 100
    assert oracle.lbp_code_window(w) == 0
    w = np.full(9, 65534)
    w[4] = 65535
    assert oracle.lbp_code_window(w) == 0
    w = np.full(9, 3)
    w[4] = 0
    assert oracle.lbp_code_window(w) == 255


def test_code_range_and_equal_neighbours_all_3pow9():
    """All 3^9 = 19,683 windows over {0,1,2} (SURVEY §8c brute force): bit p set iff
    g_p >= g_c, checked through the golden Fig. 7 weights (a set bit's weight matches the
    neighbour's position).  Every window goes through the oracle's map routine (the windows
    side by side in 3x3 blocks of one strip, codes read at the block centres) and every 7th
    also through the single-window entry point."""
    _, _, weights, _ = _golden_fig7()
    grid = np.array(np.meshgrid(*[np.arange(3)] * 9, indexing="ij")).reshape(9, -1).T
    nwin = grid.shape[0]
    assert nwin == 3 ** 9
    wins = grid.reshape(nwin, 3, 3)
    strip = np.ascontiguousarray(wins.transpose(1, 0, 2).reshape(3, 3 * nwin)).astype(np.uint8)
    codes = oracle.lbp_map_u8(strip)[0, 3 * np.arange(nwin)].astype(np.int64)
    ge = (wins >= wins[:, 1:2, 1:2]).astype(np.int64)
    ge[:, 1, 1] = 0
    expect = (ge * weights[None, :, :]).reshape(nwin, 9).sum(1)
    assert np.array_equal(codes, expect)
    assert codes.min() >= 0 and codes.max() <= 255
    for k in range(0, nwin, 7):
        assert oracle.lbp_code_window(wins[k]) == expect[k]


def test_map_rotation_and_flip_metamorphic():
    """Rotating the image 90 deg CW rotates every code left by 2 bits (the Fig. 7 positions go
    clockwise); CCW -> rotl 6; a horizontal flip permutes bits 0<->2, 3<->7, 4<->6."""
    rng = np.random.default_rng(5)
    img = rng.integers(0, 6, (23, 17)).astype(np.uint8)  # many ties
    m = oracle.lbp_map_u8(img).astype(np.int64)
    m_cw = oracle.lbp_map_u8(np.ascontiguousarray(np.rot90(img, -1))).astype(np.int64)
    assert np.array_equal(m_cw, rotl8(np.rot90(m, -1), 2))
    m_ccw = oracle.lbp_map_u8(np.ascontiguousarray(np.rot90(img, 1))).astype(np.int64)
    assert np.array_equal(m_ccw, rotl8(np.rot90(m, 1), 6))
    m_fl = oracle.lbp_map_u8(np.ascontiguousarray(img[:, ::-1])).astype(np.int64)
    perm = {0: 2, 2: 0, 3: 7, 7: 3, 4: 6, 6: 4, 1: 1, 5: 5}
    flipped = np.zeros_like(m)
    for p, q in perm.items():
        flipped |= ((m[:, ::-1] >> p) & 1) << q
    assert np.array_equal(m_fl, flipped)


def test_map_monotone_invariance():
    """S:408 / P:111: for strictly increasing phi, codes(phi(img)) = codes(img)."""
    rng = np.random.default_rng(11)
    img = rng.integers(0, 64, (31, 29)).astype(np.uint8)
    phi = np.sort(rng.choice(256, 64, replace=False)).astype(np.uint8)
    assert np.array_equal(oracle.lbp_map_u8(phi[img]), oracle.lbp_map_u8(img))


# --------------------------------------------------------------------------- uniform bins

def test_uniform_table_closed_form():
    """Uniform codes = {0, 255} U {circular runs rotl(2^k - 1, r)}: 2 + 8*7 = 58 codes, 59 bins."""
    table, n_uniform = oracle.uniform_table()
    assert n_uniform == 58
    runs = {0, 255} | {int(rotl8((1 << k) - 1, r)) for k in range(1, 8) for r in range(8)}
    assert len(runs) == 58
    uniform = {c for c in range(256) if table[c] < 58}
    assert uniform == runs
    assert sorted(table[sorted(runs)].tolist()) == list(range(58))
    # ascending-code numbering; values from SURVEY appendix
    assert [table[c] for c in (0, 1, 127, 241, 254, 255, 85, 170)] == [0, 1, 28, 48, 56, 57, 58, 58]
    assert all(table[sorted(runs)][i] < table[sorted(runs)][i + 1] for i in range(57))
    # rotation maps uniform to uniform
    for c in runs:
        assert table[int(rotl8(c, 3))] < 58


# --------------------------------------------------------------------------- histograms

def _cell_index(n_px, K):
    """Inverse of the floor partition (a different formula from the oracle's block loop):
    pixel j is in cell floor(((j+1)*K - 1) / n_px)."""
    j = np.arange(n_px)
    return ((j + 1) * K - 1) // n_px


def _valid_mask(depth, dmin, dmax):
    return (depth != 0) & (depth >= dmin) & (depth <= dmax)


@pytest.mark.parametrize("H,W,K", [(64, 64, (8, 8)), (128, 128, (8, 8)), (37, 53, (5, 3)),
                                   (20, 131, (7, 9)), (9, 9, (7, 1))])
@pytest.mark.parametrize("bins", [59, 256])
def test_cell_sums_equal_valid_counts(H, W, K, bins):
    """J.north_star invariant: each cell histogram sums to its count of valid depth-masked px."""
    grey, depth = synthgen.face_crops(3, H, W, seed=7)
    kx, ky = K
    desc = oracle.lbp_extract(grey, depth, synthgen.full_rois(3, H, W), 600, 1400, kx, ky, bins)
    cx, cy = _cell_index(W - 2, kx), _cell_index(H - 2, ky)
    for n in range(3):
        valid = _valid_mask(depth[n, 1:-1, 1:-1], 600, 1400)
        expect = np.zeros((ky, kx), np.int64)
        np.add.at(expect, (cy[:, None].repeat(W - 2, 1), cx[None, :].repeat(H - 2, 0)), valid)
        got = desc[n].reshape(ky, kx, bins).sum(-1)
        assert np.array_equal(got, expect)


def test_no_mask_total_and_spec_value():
    """200x200 ROI, 1x1 grid, 256 bins, no mask -> total 39204 = 198^2."""
    grey, _ = synthgen.face_crops(1, 200, 200, seed=3)
    desc = oracle.lbp_extract(grey, None, synthgen.full_rois(1, 200, 200), 0, 65535, 1, 1, 256)
    assert int(desc.sum()) == 39204


@pytest.mark.parametrize("bins,bin_const", [(59, 57), (256, 255)])
def test_constant_image_single_code(bins, bin_const):
    """Constant image -> every code 255 -> one bin per cell, count = cell valid count."""
    grey, depth = synthgen.face_crops(2, 64, 64, dist="constant")
    desc = oracle.lbp_extract(grey, depth, synthgen.full_rois(2, 64, 64), 600, 1400, 8, 8, bins)
    h = desc.reshape(2, 64, bins)
    assert np.array_equal(h.sum(-1), h[:, :, bin_const])
    assert int(h.sum()) == 2 * 62 * 62


def test_refinement_and_partition():
    """(16,16) summed in 2x2 groups == (8,8) when the interior is divisible (130 -> 128);
    S:378: sum over cells == the 1x1 histogram, for any grid."""
    grey, depth = synthgen.face_crops(2, 130, 130, seed=9)
    rois = synthgen.full_rois(2, 130, 130)
    d16 = oracle.lbp_extract(grey, depth, rois, 600, 1400, 16, 16, 59).reshape(2, 8, 2, 8, 2, 59)
    d8 = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 59).reshape(2, 8, 8, 59)
    assert np.array_equal(d16.sum(axis=(2, 4)), d8)
    d1 = oracle.lbp_extract(grey, depth, rois, 600, 1400, 1, 1, 256)
    for kx, ky in [(3, 7), (5, 5), (13, 2)]:
        dk = oracle.lbp_extract(grey, depth, rois, 600, 1400, kx, ky, 256)
        assert np.array_equal(dk.reshape(2, -1, 256).sum(1), d1)


def test_uniform_fold_of_256():
    """59-bin descriptor = the 256-bin one folded through the (pinned) uniform table."""
    grey, depth = synthgen.face_crops(2, 48, 40, seed=1)
    rois = synthgen.full_rois(2, 48, 40)
    table, _ = oracle.uniform_table()
    d256 = oracle.lbp_extract(grey, depth, rois, 600, 1400, 4, 3, 256).reshape(2, 12, 256)
    d59 = oracle.lbp_extract(grey, depth, rois, 600, 1400, 4, 3, 59).reshape(2, 12, 59)
    fold = np.zeros_like(d59, dtype=np.int64)
    for c in range(256):
        fold[:, :, table[c]] += d256[:, :, c]
    assert np.array_equal(fold, d59)


def test_mask_special_cases():
    """Window [1,65535] on zero-free depth == depth=NULL; empty window -> zero descriptor;
    depth 0 is invalid even with dmin = 0; only the CENTRE pixel is gated."""
    grey, depth = synthgen.face_crops(2, 40, 40, seed=2)
    rois = synthgen.full_rois(2, 40, 40)
    dz = np.maximum(depth, 1)
    a = oracle.lbp_extract(grey, dz, rois, 1, 65535, 3, 3, 59)
    b = oracle.lbp_extract(grey, None, rois, 0, 0, 3, 3, 59)
    assert np.array_equal(a, b)
    assert oracle.lbp_extract(grey, depth, rois, 1, 1, 3, 3, 59).sum() == 0
    zero = np.zeros_like(depth)
    assert oracle.lbp_extract(grey, zero, rois, 0, 65535, 3, 3, 59).sum() == 0
    # only the centre: invalidate every pixel except one interior centre -> total 1
    g = np.arange(25, dtype=np.uint8).reshape(1, 5, 5)
    d = np.zeros((1, 5, 5), np.uint16)
    d[0, 2, 2] = 1000
    one = oracle.lbp_extract(g, d, [[0, 0, 0, 5, 5]], 600, 1400, 1, 1, 256)
    assert int(one.sum()) == 1


def test_tiny_crops_brute_force_all_grids():
    """3x3..6x6 ROIs with every grid 1..W' x 1..H' == per-pixel code map + inverse
    cell formula (brute force)."""
    rng = np.random.default_rng(4)
    for H in range(3, 7):
        for W in range(3, 7):
            grey = rng.integers(0, 4, (1, H, W)).astype(np.uint8)
            depth = rng.integers(0, 3, (1, H, W)).astype(np.uint16) * 500
            codes = oracle.lbp_map_u8(grey[0]).astype(np.int64)
            valid = _valid_mask(depth[0, 1:-1, 1:-1], 400, 600)
            for kx in range(1, W - 1):
                for ky in range(1, H - 1):
                    desc = oracle.lbp_extract(grey, depth, [[0, 0, 0, W, H]], 400, 600, kx, ky, 256)
                    expect = np.zeros((ky, kx, 256), np.int64)
                    cx, cy = _cell_index(W - 2, kx), _cell_index(H - 2, ky)
                    for i in range(H - 2):
                        for j in range(W - 2):
                            if valid[i, j]:
                                expect[cy[i], cx[j], codes[i, j]] += 1
                    assert np.array_equal(desc.reshape(ky, kx, 256), expect)


# --------------------------------------------------------------------------- ROI semantics

def test_roi_clamp_equals_intersection():
    """an ROI sticking out of the image is clamped to the intersection."""
    grey, depth = synthgen.face_crops(2, 50, 60, seed=8)
    out = oracle.lbp_extract(grey, depth, [[1, -5, 40, 30, 30]], 600, 1400, 3, 2, 59)
    ref = oracle.lbp_extract(grey, depth, [[1, 0, 40, 25, 10]], 600, 1400, 3, 2, 59)
    assert np.array_equal(out, ref)
    # every side, on noise with every pixel counted (no all-masked / all-equal descriptors)
    rng = np.random.default_rng(3)
    g = rng.integers(0, 256, (2, 50, 60), dtype=np.uint8)
    d = np.full((2, 50, 60), 1000, np.uint16)
    cases = [([1, -5, 3, 30, 30], [1, 0, 3, 25, 30]),     # left
             ([0, 7, -9, 20, 30], [0, 7, 0, 20, 21]),     # top
             ([1, 45, 10, 40, 12], [1, 45, 10, 15, 12]),  # right
             ([0, 4, 41, 20, 40], [0, 4, 41, 20, 9]),     # bottom
             ([1, -3, -4, 80, 90], [1, 0, 0, 60, 50])]    # all four
    for roi, inter in cases:
        for dep in (None, d):
            a = oracle.lbp_extract(g, dep, [roi], 600, 1400, 3, 2, 59)
            r = oracle.lbp_extract(g, dep, [inter], 600, 1400, 3, 2, 59)
            assert a.sum() > 0 and np.array_equal(a, r), (roi, dep is None)


def test_roi_error_statuses():
    """S:86 empty -> E_ROI; S:365 <3 px -> E_ROI; S:372 grid > interior -> E_GRID;
    u16 overflow -> E_OVERFLOW; failed rows are zero-filled."""
    grey = np.full((2, 300, 300), 9, np.uint8)
    rois = [[0, 400, 0, 10, 10],     # outside
            [0, 0, 0, 2, 50],        # too narrow
            [5, 0, 0, 10, 10],       # bad image index
            [0, 0, 0, 6, 6],         # 4x4 interior, 5x5 grid
            [0, 0, 0, 260, 260],     # 258^2 > 65535 in one cell
            [0, 0, 0, 257, 257],     # 255^2 fits
            [1, 298, 298, 50, 50],   # clamps to 2x2 -> E_ROI
            [1, 0, 0, 258, 258]]     # 256^2 = 65536 just overflows u16
    desc, st = oracle.lbp_extract(grey, None, rois, 0, 65535, 1, 1, 59, return_status=True)
    assert st.tolist() == [-2, -2, -2, 0, -4, 0, -2, -4]
    assert desc[[0, 1, 2, 4, 6, 7]].sum() == 0
    desc, st = oracle.lbp_extract(grey, None, [[0, 0, 0, 6, 6]], 0, 65535, 5, 5, 59,
                                  return_status=True)
    assert st.tolist() == [-3] and desc.sum() == 0
    assert int(oracle.lbp_extract(grey, None, [[0, 0, 0, 257, 257]], 0, 65535, 1, 1, 59)[0, 57]) == 65025


def test_argument_validation():
    L = oracle.lib()
    g = np.zeros((1, 8, 8), np.uint8)
    r = np.array([[0, 0, 0, 8, 8]], np.int32)
    out = np.zeros(59 * 4, np.uint16)
    P = lambda a: a.ctypes.data

    def call(bins=59, cx=2, cy=2, dmin=0, dmax=10, n=1, desc=out, pitch=8):
        return L.oracle_lbp_extract(P(g), None, 1, 8, 8, pitch, 8, 64, 64, P(r), n, dmin, dmax,
                                    cx, cy, bins, None if desc is None else P(desc), None)
    assert call() == 0
    assert call(bins=60) == -1
    assert call(cx=0) == -1
    assert call(dmin=11) == -1
    assert call(desc=None) == -1
    assert call(pitch=7) == -1
    assert call(n=0, desc=None) == 0


# --------------------------------------------------------------------------- SVM decision

def test_svm_closed_forms():
    """One-hot W rows -> the bin count exactly; all-ones W -> valid count + b (P:142 hyperplane)."""
    grey, depth = synthgen.face_crops(4, 64, 64, seed=12)
    desc = oracle.lbp_extract(grey, depth, synthgen.full_rois(4, 64, 64), 600, 1400, 8, 8, 59)
    D = desc.shape[1]
    picks = [0, 57, 58, 1000, D - 1]
    W = np.zeros((len(picks) + 1, D), np.float32)
    for c, d in enumerate(picks):
        W[c, d] = 1.0
    W[-1] = 1.0
    b = np.array([0, 0.5, -2, 0, 0, 3.25], np.float32)
    s, _, _ = oracle.svm_score(desc, W, b)
    for c, d in enumerate(picks):
        assert np.array_equal(s[:, c], desc[:, d].astype(np.float32) + b[c])
    assert np.array_equal(s[:, -1], desc.sum(1).astype(np.float32) + b[-1])


def test_svm_integer_weights_exact():
    """Integer W (|w| <= 1000) and integer b: every partial sum < 2^24 so the result is exact."""
    grey, depth = synthgen.face_crops(6, 128, 128, seed=13)
    desc = oracle.lbp_extract(grey, depth, synthgen.full_rois(6, 128, 128), 600, 1400, 8, 8, 59)
    rng = np.random.default_rng(3)
    W = rng.integers(-1000, 1001, (10, desc.shape[1])).astype(np.float32)
    b = rng.integers(-50, 51, 10).astype(np.float32)
    s, lab, top = oracle.svm_score(desc, W, b)
    exact = desc.astype(np.int64) @ W.astype(np.int64).T + b.astype(np.int64)
    assert np.array_equal(s.astype(np.int64), exact)
    assert np.array_equal(lab, np.argmax(exact, axis=1))


def test_svm_random_within_fp32_rounding_of_exact():
    """Random W ~ N(0, 2^-8): oracle score within 1 fp32 ulp of the EXACT rational sum
    (math.fsum = correctly rounded double of the exact sum, then rounded to fp32)."""
    grey, depth = synthgen.face_crops(3, 128, 128, seed=14)
    desc = oracle.lbp_extract(grey, depth, synthgen.full_rois(3, 128, 128), 600, 1400, 8, 8, 59)
    W, b = synthgen.svm_weights(7, desc.shape[1], seed=1)
    s, _, _ = oracle.svm_score(desc, W, b)
    for n in range(3):
        for c in range(7):
            terms = [float(W[c, d]) * int(desc[n, d]) for d in range(desc.shape[1])]
            # each product is exact in double (24-bit x 16-bit)
            assert Fraction(terms[5]) == Fraction(float(W[c, 5])) * int(desc[n, 5])
            exact = np.float32(math.fsum(terms + [float(b[c])]))
            assert abs(float(s[n, c]) - float(exact)) <= float(np.spacing(np.abs(exact)))


def test_svm_ties_and_reject():
    """ties -> lowest class index; top < threshold -> -1; +inf rejects all."""
    desc = np.array([[1, 2, 3], [0, 0, 0]], np.uint16)
    W = np.array([[1, 1, 1], [1, 1, 1], [0, 0, 3]], np.float32)
    b = np.array([0, 0, -3], np.float32)
    s, lab, top = oracle.svm_score(desc, W, b)
    assert lab.tolist() == [0, 0]
    assert top.tolist() == [6.0, 0.0]
    _, lab, _ = oracle.svm_score(desc, W, b, reject_threshold=3.0)
    assert lab.tolist() == [0, -1]
    _, lab, _ = oracle.svm_score(desc, W, b, reject_threshold=float("inf"))
    assert lab.tolist() == [-1, -1]
    # the boundary: a top score EQUAL to the threshold is kept (strict "<")
    _, lab, _ = oracle.svm_score(desc, W, b, reject_threshold=6.0)
    assert lab.tolist() == [0, -1]
    _, lab, _ = oracle.svm_score(desc, W, b, reject_threshold=float(np.nextafter(np.float32(6.0),
                                                                                 np.float32(7.0))))
    assert lab.tolist() == [-1, -1]
