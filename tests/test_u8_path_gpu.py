"""The compact recognition path on the device (R21, R22):
lbp_extract_u8 (the TMA kernel's epilogue writes u8 rows + per-row records of the entries above
255) and svm_score_u8 (the INT8 tensor-core scorer reading those bytes by TMA), against the
oracle: the compact descriptor must decode to exactly the oracle's u16 descriptor (bit-exact,
every row), and the scores / labels / top scores must satisfy R13 / R14 (oracle/tolerance.py).

Exception cases: crops with k uniform 16x16 cells (a constant 18x18 patch covering the cell and
its 1-px halo makes all 256 codes of the cell equal -> one count of 256), k = 1..3 (records
in shared memory), constant crops (64 exceptions per row: the scorer's fp64 row path) and a
tile with more than 32 distinct exception columns (W not staged: fp64 rows)."""
import numpy as np
import pytest
import torch

import oracle
import synthgen
from oracle.tolerance import check_svm

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def lb():
    import paper_1504_01883_b200 as m
    return m


FULL = (1, 2, 3, 5, 6, 7)  # cell rows / columns of 16 interior pixels (floor partition of 126)


def _patch_cells(grey, depth, idx, cells, value=90):
    """Cell (cy, cx) of crop idx uniform: interior rows [floor(126 cy / 8), +16) are image rows
    1 + ..., so an 18x18 constant patch from image row / column floor(126 c / 8) covers the
    cell and its 1-px halo: every code of the cell is 255 -> one count of 256 (cy, cx in
    FULL)."""
    for cy, cx in cells:
        y0, x0 = (cy * 126) // 8, (cx * 126) // 8
        grey[idx, y0:y0 + 18, x0:x0 + 18] = value
        depth[idx, y0:y0 + 18, x0:x0 + 18] = 1000


def _inputs(n, H=128, seed=3, exc_every=0, const_every=0, many_cols=False):
    g, d = synthgen.face_crops(n, H, H, seed=seed)
    rng = np.random.default_rng(seed)
    for i in range(n):
        if const_every and i % const_every == 0:
            g[i] = 77
            d[i] = 1000
        elif exc_every and i % exc_every == 1:
            k = 1 + i % 3
            if many_cols:  # spread over many cells -> many distinct columns in a tile
                cells = [(int(rng.choice(FULL)), int(rng.choice(FULL))) for _ in range(k)]
            else:
                cells = [(2, 3), (5, 1), (6, 6)][:k]
            _patch_cells(g, d, i, cells, value=int(rng.integers(20, 230)))
    return g, d


def _to_dev(g, d, rois):
    return (torch.from_numpy(g).to(DEV),
            torch.from_numpy(d.view(np.int16)).to(DEV).view(torch.uint16),
            torch.from_numpy(rois).to(DEV))


def _decode(cd):
    """u16 descriptor from the compact form (host-side, independent of the CUDA unpack)."""
    packed = cd.packed.cpu().numpy().astype(np.uint16)
    n_exc = cd.exc_n.cpu().numpy()
    exc = cd.exc.cpu().numpy().view(np.uint32)
    out = packed.copy()
    for i in np.nonzero(n_exc)[0]:
        for k in range(min(int(n_exc[i]), exc.shape[1])):
            r = int(exc[i, k])
            out[i, r >> 16] = r & 0xFFFF
    return out, n_exc


def _check_compact(cd, ref):
    got, n_exc = _decode(cd)
    bad = np.nonzero((got != ref).any(1))[0]
    assert bad.size == 0, f"rows {bad[:10]} differ from the oracle"
    assert np.array_equal(n_exc, (ref > 255).sum(1))
    assert np.array_equal(cd.packed.cpu().numpy(), (ref & 255).astype(np.uint8))


@pytest.mark.parametrize("n,exc_every,const_every", [(301, 0, 0), (400, 4, 0), (300, 5, 7),
                                                      (2000, 50, 0)])
def test_extract_u8_fast_path(lb, n, exc_every, const_every):
    g, d = _inputs(n, exc_every=exc_every, const_every=const_every)
    rois = synthgen.full_rois(n, 128, 128)
    grey, depth, r = _to_dev(g, d, rois)
    st = torch.full((n,), -99, dtype=torch.int32, device=DEV)
    cd = lb.lbp_extract_u8(grey, depth, r, 600, 1400, 8, 8, 59, roi_status=st)
    torch.cuda.synchronize()
    ref = oracle.lbp_extract(g, d, rois, 600, 1400, 8, 8, 59)
    if exc_every or const_every:
        assert (ref > 255).any()
    _check_compact(cd, ref)
    assert (st.cpu().numpy() == 0).all()


def test_extract_u8_generic_rois_in_fast_kernel(lb):
    """ROIs off the TMA path (clamped, odd sizes, outside) inside the persistent kernel: the
    generic code path counts into the group's counters and stages the u8 row the same way."""
    n_img, n = 40, 400
    g, d = _inputs(n_img, exc_every=3)
    rois = synthgen.random_rois(n, n_img, 128, 128, seed=4)
    rois[::5] = synthgen.full_rois(n, 128, 128)[::5] % [n_img, 1, 1, 1000, 1000]
    grey, depth, r = _to_dev(g, d, rois)
    st = torch.full((n,), -99, dtype=torch.int32, device=DEV)
    cd = lb.lbp_extract_u8(grey, depth, r, 600, 1400, 8, 8, 59, roi_status=st)
    torch.cuda.synchronize()
    ref, st_ref = oracle.lbp_extract(g, d, rois, 600, 1400, 8, 8, 59, return_status=True)
    _check_compact(cd, ref)
    assert np.array_equal(st.cpu().numpy(), st_ref)
    assert (st_ref != 0).any() and (st_ref == 0).any()


@pytest.mark.parametrize("n,H,cells,bins", [(20, 128, 8, 59), (150, 64, 4, 59),
                                            (37, 128, 8, 256), (3, 200, 2, 59)])
def test_extract_u8_packed_fallback(lb, n, H, cells, bins):
    """Off the TMA kernel: u16 extraction into a scratch, then the per-row pack kernel (200x200
    with 2x2 cells has counts up to 99^2 -> several records per row)."""
    g, d = synthgen.face_crops(n, H, H, seed=8)
    if H == 200:
        g[:, :120, :120] = 50
        d[:, :120, :120] = 1000
    rois = synthgen.full_rois(n, H, H)
    grey, depth, r = _to_dev(g, d, rois)
    cd = lb.lbp_extract_u8(grey, depth, r, 600, 1400, cells, cells, bins)
    torch.cuda.synchronize()
    ref = oracle.lbp_extract(g, d, rois, 600, 1400, cells, cells, bins)
    if H == 200:
        assert (ref > 255).sum(1).max() > 1
    _check_compact(cd, ref)


def _svm_u8(lb, cd, W, b, prepared=True, want_scores=True, reject=float("-inf")):
    Wt, bt = torch.from_numpy(W).to(DEV), torch.from_numpy(b).to(DEV)
    prep = lb.svm_prepare_u8(Wt) if prepared else None
    s, lab, top = lb.svm_score_u8(cd, Wt, bt, prepared=prep, want_scores=want_scores,
                                  reject_threshold=reject)
    torch.cuda.synchronize()
    return (None if s is None else s.cpu().numpy()), lab.cpu().numpy(), top.cpu().numpy()


@pytest.mark.parametrize("C", [1, 2, 10, 100, 102, 103, 250, 1000])
def test_svm_u8_tensor_core(lb, C):
    n = 300
    g, d = _inputs(n, seed=C, exc_every=6, const_every=0)
    rois = synthgen.full_rois(n, 128, 128)
    grey, depth, r = _to_dev(g, d, rois)
    cd = lb.lbp_extract_u8(grey, depth, r, 600, 1400, 8, 8, 59)
    ref = oracle.lbp_extract(g, d, rois, 600, 1400, 8, 8, 59)
    W, b = synthgen.svm_weights(C, 3776, seed=C)
    s, lab, top = _svm_u8(lb, cd, W, b)
    s_ref, lab_ref, _ = oracle.svm_score(ref, W, b)
    ok, detail = check_svm(ref, W, b, s_ref, lab_ref, lab, s_gpu=s, top_gpu=top)
    assert ok, detail
    # label-only mode (4 digits + per-row proof + exact fix-up of unproven rows)
    _, lab2, top2 = _svm_u8(lb, cd, W, b, want_scores=False)
    ok, detail = check_svm(ref, W, b, s_ref, lab_ref, lab2, top_gpu=top2)
    assert ok, detail
    assert (lab2 >= 0).all()  # no row left unresolved


@pytest.mark.parametrize("case", ["constant", "many_columns", "no_prepare", "small_n"])
def test_svm_u8_exception_paths(lb, case):
    n = 100 if case == "small_n" else 600
    g, d = _inputs(n, seed=11, exc_every=2 if case == "many_columns" else 9,
                   const_every=5 if case == "constant" else 0, many_cols=case == "many_columns")
    rois = synthgen.full_rois(n, 128, 128)
    grey, depth, r = _to_dev(g, d, rois)
    cd = lb.lbp_extract_u8(grey, depth, r, 600, 1400, 8, 8, 59)
    ref = oracle.lbp_extract(g, d, rois, 600, 1400, 8, 8, 59)
    assert (ref > 255).any()
    W, b = synthgen.svm_weights(100, 3776, seed=7)
    s, lab, top = _svm_u8(lb, cd, W, b, prepared=case != "no_prepare")
    s_ref, lab_ref, _ = oracle.svm_score(ref, W, b)
    ok, detail = check_svm(ref, W, b, s_ref, lab_ref, lab, s_gpu=s, top_gpu=top)
    assert ok, detail


def test_svm_u8_integer_weights_bitexact(lb):
    """Integer W, b: every path is exact -> bit-exact scores, labels, top scores."""
    n = 260
    g, d = _inputs(n, seed=2, exc_every=5, const_every=13)
    rois = synthgen.full_rois(n, 128, 128)
    grey, depth, r = _to_dev(g, d, rois)
    cd = lb.lbp_extract_u8(grey, depth, r, 600, 1400, 8, 8, 59)
    ref = oracle.lbp_extract(g, d, rois, 600, 1400, 8, 8, 59)
    rng = np.random.default_rng(1)
    W = rng.integers(-1000, 1001, (100, 3776)).astype(np.float32)
    b = rng.integers(-50, 51, 100).astype(np.float32)
    s_ref, lab_ref, top_ref = oracle.svm_score(ref, W, b)
    for prepared in (True, False):
        s, lab, top = _svm_u8(lb, cd, W, b, prepared=prepared)
        assert np.array_equal(s, s_ref) and np.array_equal(lab, lab_ref)
        assert np.array_equal(top, top_ref)


@pytest.mark.parametrize("C", [3, 100, 1000])
def test_svm_u8_label_mode_fixup(lb, C):
    """Label-only mode on rows its proof cannot settle: exact ties between two classes (every
    row), and a reject threshold equal to some rows' exact top score -- every such row goes to
    the fix-up kernel and must come back equal to the oracle (ties -> lower class)."""
    n = 300
    g, d = _inputs(n, seed=5, exc_every=7)
    rois = synthgen.full_rois(n, 128, 128)
    grey, depth, r = _to_dev(g, d, rois)
    cd = lb.lbp_extract_u8(grey, depth, r, 600, 1400, 8, 8, 59)
    ref = oracle.lbp_extract(g, d, rois, 600, 1400, 8, 8, 59)
    W, b = synthgen.svm_weights(C, 3776, seed=C + 1)
    W[C - 1] = W[C // 2]
    b[C - 1] = b[C // 2] = 1e4  # classes C//2 and C-1 tie at the top of every row
    s_ref, lab_ref, top_ref = oracle.svm_score(ref, W, b)
    _, lab, top = _svm_u8(lb, cd, W, b, want_scores=False)
    assert np.array_equal(lab, lab_ref) and (lab == C // 2).all()
    assert np.array_equal(top, top_ref)
    # reject threshold at the exact top score of rows 0..9 (ties with the threshold)
    W2, b2 = synthgen.svm_weights(C, 3776, seed=C + 2)
    s2, lab2r, top2r = oracle.svm_score(ref, W2, b2)
    for k in range(3):
        rej = float(top2r[k])
        _, l2, t2 = _svm_u8(lb, cd, W2, b2, want_scores=False, reject=rej)
        _, l2r, _ = oracle.svm_score(ref, W2, b2, reject_threshold=rej)
        assert l2[k] == l2r[k]
        ok, detail = check_svm(ref, W2, b2, s2, l2r, l2, top_gpu=t2)
        assert ok, detail


def test_svm_u8_ties_reject_and_bad_model(lb):
    n = 256
    g, d = _inputs(n, seed=4)
    rois = synthgen.full_rois(n, 128, 128)
    grey, depth, r = _to_dev(g, d, rois)
    cd = lb.lbp_extract_u8(grey, depth, r, 600, 1400, 8, 8, 59)
    W, b = synthgen.svm_weights(4, 3776, seed=3)
    W[2] = W[1]
    b[2] = b[1] = 1e4
    _, lab, top = _svm_u8(lb, cd, W, b)
    assert (lab == 1).all()
    _, lab, _ = _svm_u8(lb, cd, W, b, reject=float("inf"))
    assert (lab == -1).all()
    # a workspace prepared for another W: refused on the device (LBP_LABEL_BAD_MODEL, NaN)
    Wt, bt = torch.from_numpy(W).to(DEV), torch.from_numpy(b).to(DEV)
    other = lb.svm_prepare_u8(Wt + 1.0)
    s, lab, top = lb.svm_score_u8(cd, Wt, bt, prepared=other)
    torch.cuda.synchronize()
    assert (lab.cpu().numpy() == -2).all() and torch.isnan(top).all()


def test_svm_u8_fullsize_sampled(lb):
    """The bench's configuration (16,384 crops, C = 100, face crops with ~1 % exception rows):
    every descriptor row decoded bit-exact; scores of 512 sampled rows within R13, all labels
    on the clear rows of that sample equal to the oracle's."""
    n = 16384
    grey, depth = synthgen.gpu_face_crops(n, 128, 128, seed=42, device=DEV)
    rois = torch.from_numpy(synthgen.full_rois(n, 128, 128)).to(DEV)
    cd = lb.lbp_extract_u8(grey, depth, rois, 600, 1400, 8, 8, 59)
    W, b = synthgen.svm_weights(100, 3776, seed=42)
    s, lab, top = _svm_u8(lb, cd, W, b)
    idx = np.unique(np.linspace(0, n - 1, 512).astype(np.int64))
    ti = torch.from_numpy(idx).to(DEV)
    g = grey[ti].cpu().numpy()
    dd = depth.view(torch.int16)[ti].cpu().numpy().view(np.uint16)
    ref = oracle.lbp_extract(g, dd, synthgen.full_rois(len(idx), 128, 128), 600, 1400, 8, 8, 59)
    got, _ = _decode(lb.CompactDesc(cd.packed[ti], cd.exc_n[ti], cd.exc[ti]))
    assert np.array_equal(got, ref)
    s_ref, lab_ref, _ = oracle.svm_score(ref, W, b)
    ok, detail = check_svm(ref, W, b, s_ref, lab_ref, lab[idx], s_gpu=s[idx], top_gpu=top[idx])
    assert ok, detail
