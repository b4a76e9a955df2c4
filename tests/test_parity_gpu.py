"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Descriptors and ROI statuses must be bit-exact; SVM scores within 1e-5 relative
(J.north_star; tests/parity_util.py) and labels identical away from ties.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synthgen
from parity_util import labels_agree_away_from_ties, svm_tolerance_ok

pytestmark = pytest.mark.gpu

DEV = "cuda"


@pytest.fixture(scope="module")
def lb():
    import paper_1504_01883_b200 as lb
    lb.lbpfused.lib()
    return lb


def _gpu_extract(lb, grey, depth, rois, dmin, dmax, kx, ky, bins, with_status=True):
    g = torch.from_numpy(np.ascontiguousarray(grey)).to(DEV)
    d = None if depth is None else torch.from_numpy(np.ascontiguousarray(depth).view(np.int16)).to(DEV).view(torch.uint16)
    r = torch.from_numpy(np.ascontiguousarray(rois, dtype=np.int32)).to(DEV)
    st = torch.full((r.shape[0],), 123, dtype=torch.int32, device=DEV)
    out = lb.lbp_fused_extract(g, d, r, dmin, dmax, kx, ky, bins,
                               roi_status=st if with_status else None)
    torch.cuda.synchronize()
    return out.cpu().view(torch.int16).numpy().view(np.uint16), st.cpu().numpy()


def _check(lb, grey, depth, rois, dmin, dmax, kx, ky, bins):
    got, st = _gpu_extract(lb, grey, depth, rois, dmin, dmax, kx, ky, bins)
    ref, st_ref = oracle.lbp_extract(grey, depth, rois, dmin, dmax, kx, ky, bins, return_status=True)
    assert np.array_equal(st, st_ref)
    bad = np.nonzero((got != ref).any(1))[0]
    assert bad.size == 0, f"{bad.size} rows differ, first {bad[:5]}"


@pytest.mark.parametrize("bins", [59, 256])
@pytest.mark.parametrize("dist", ["face", "constant", "noise"])
def test_crops_128_bitexact(lb, bins, dist):
    # >= 148 ROIs: the persistent TMA kernels (smaller batches take the band kernel)
    grey, depth = synthgen.face_crops(160, 128, 128, seed=21, dist=dist)
    _check(lb, grey, depth, synthgen.full_rois(160, 128, 128), 600, 1400, 8, 8, bins)
    _check(lb, grey[:20], depth[:20], synthgen.full_rois(20, 128, 128), 600, 1400, 8, 8, bins)


def test_crop_64_config1(lb):
    grey, depth = synthgen.face_crops(1, 64, 64, seed=1)
    _check(lb, grey, depth, synthgen.full_rois(1, 64, 64), 600, 1400, 8, 8, 59)


@pytest.mark.parametrize("bins", [59, 256])
def test_no_depth_mask(lb, bins):
    grey, _ = synthgen.face_crops(150, 128, 128, seed=2)  # TMA kernels without depth
    _check(lb, grey, None, synthgen.full_rois(150, 128, 128), 0, 0, 8, 8, bins)
    _check(lb, grey[:8], None, synthgen.full_rois(8, 128, 128), 0, 0, 8, 8, bins)


@pytest.mark.parametrize("H,W,kx,ky", [(37, 53, 5, 3), (20, 131, 7, 9), (9, 9, 7, 1),
                                       (130, 130, 16, 16), (200, 200, 1, 1), (66, 70, 8, 8)])
@pytest.mark.parametrize("bins", [59, 256])
def test_ragged_random_rois(lb, H, W, kx, ky, bins):
    grey, depth = synthgen.face_crops(5, H, W, seed=H * W)
    rois = synthgen.random_rois(40, 5, H, W, seed=kx * 31 + ky, min_size=1)
    rois[0] = (0, 0, 0, W, H)
    _check(lb, grey, depth, rois, 600, 1400, kx, ky, bins)


def test_tiny_rois_every_grid(lb):
    grey, depth = synthgen.face_crops(1, 8, 8, seed=3, dist="noise")
    for w in range(1, 8):
        for h in range(1, 8):
            for kx in range(1, 6):
                for ky in range(1, 6):
                    _check(lb, grey, depth, [[0, 1, 0, w, h]], 0, 65535, kx, ky, 256)


def test_large_grid_chunked(lb):
    """16x16 cells x 256 bins = 65536 counters: more than one shared-memory chunk."""
    grey, depth = synthgen.face_crops(3, 200, 200, seed=4)
    _check(lb, grey, depth, synthgen.full_rois(3, 200, 200), 600, 1400, 16, 16, 256)
    _check(lb, grey, depth, synthgen.full_rois(3, 200, 200), 600, 1400, 40, 30, 59)


def test_error_rois_and_overflow(lb):
    grey = np.full((2, 300, 300), 9, np.uint8)
    rois = [[0, 400, 0, 10, 10], [0, 0, 0, 2, 50], [5, 0, 0, 10, 10], [0, 0, 0, 6, 6],
            [0, 0, 0, 260, 260], [0, 0, 0, 257, 257], [1, 298, 298, 50, 50], [1, 0, 0, 258, 258],
            [-1, 0, 0, 10, 10], [0, -10, -10, 5, 5], [1, 290, 290, 1000, 1000]]
    _check(lb, grey, None, rois, 0, 65535, 1, 1, 59)
    _check(lb, grey, None, rois, 0, 65535, 5, 5, 256)


def test_depth_window_edges(lb):
    grey, depth = synthgen.face_crops(4, 64, 64, seed=5)
    rois = synthgen.full_rois(4, 64, 64)
    for dmin, dmax in [(0, 0), (0, 65535), (1, 1), (1000, 1000), (0, 950), (2000, 65535),
                       (65535, 65535)]:
        _check(lb, grey, depth, rois, dmin, dmax, 8, 8, 59)


def test_pitched_frames_config2(lb):
    """640x480 Kinect frames (pitched views of wider buffers) with 4 ROIs each."""
    n_frames, H, W = 3, 480, 640
    grey, depth = synthgen.face_crops(n_frames, H, W, seed=6)
    gw = np.zeros((n_frames, H, W + 64), np.uint8)
    dw = np.zeros((n_frames, H, W + 32), np.uint16)
    gw[:, :, :W] = grey
    dw[:, :, :W] = depth
    rois = []
    for f in range(n_frames):
        for k in range(4):
            rois.append([f, 40 + 150 * k + 7 * f, 100 + 20 * k, 128, 128])
    rois = np.array(rois, np.int32)
    g = torch.from_numpy(gw).to(DEV)[:, :, :W]
    d = torch.from_numpy(dw.view(np.int16)).to(DEV).view(torch.uint16)[:, :, :W]
    r = torch.from_numpy(rois).to(DEV)
    out = lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59)
    ref = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 59)
    assert np.array_equal(out.cpu().view(torch.int16).numpy().view(np.uint16), ref)


def test_fast_kernel_mixed_rois(lb):
    """8x8 grid on aligned frames -> the TMA kernel; it must also take clamped, odd-sized,
    unaligned and invalid ROIs through its internal generic path."""
    n_frames, H, W = 6, 480, 640  # 174 ROIs: the persistent TMA kernel
    grey, depth = synthgen.face_crops(n_frames, H, W, seed=16)
    rng = np.random.default_rng(7)
    rois = []
    for f in range(n_frames):
        rois += [[f, 0, 0, 128, 128], [f, 16, 32, 128, 128], [f, 3, 5, 128, 128],
                 [f, W - 100, 10, 128, 128], [f, -20, -20, 128, 128], [f, 50, 60, 100, 90],
                 [f, 10, 10, 2, 128], [f, 700, 0, 128, 128], [f, 500, 340, 140, 140]]
        for _ in range(20):
            rois.append([f, int(rng.integers(0, W - 128)), int(rng.integers(0, H - 128)), 128, 128])
    _check(lb, grey, depth, np.array(rois, np.int32), 600, 1400, 8, 8, 59)
    _check(lb, grey, depth, np.array(rois, np.int32), 600, 1400, 8, 8, 256)
    _check(lb, grey, None, np.array(rois, np.int32), 0, 0, 8, 8, 59)


def test_empty_batch(lb):
    g = torch.zeros(1, 8, 8, dtype=torch.uint8, device=DEV)
    r = torch.zeros(0, 5, dtype=torch.int32, device=DEV)
    out = lb.lbp_fused_extract(g, None, r, 0, 10, 2, 2, 59)
    assert out.shape == (0, 236)


# --------------------------------------------------------------------------- SVM

def _svm_inputs(n, C, seed):
    grey, depth = synthgen.face_crops(n, 128, 128, seed=seed)
    desc = oracle.lbp_extract(grey, depth, synthgen.full_rois(n, 128, 128), 600, 1400, 8, 8, 59)
    W, b = synthgen.svm_weights(C, desc.shape[1], seed=seed)
    return desc, W, b


def _gpu_svm(lb, desc, W, b, reject=-math.inf, prepared=False):
    d = torch.from_numpy(desc.view(np.int16)).to(DEV).view(torch.uint16)
    Wt = torch.from_numpy(W).to(DEV)
    bt = torch.from_numpy(b).to(DEV)
    prep = lb.svm_prepare(Wt) if prepared else None
    s, lab, top = lb.svm_score(d, Wt, bt, prepared=prep, reject_threshold=reject)
    torch.cuda.synchronize()
    return s.cpu().numpy(), lab.cpu().numpy(), top.cpu().numpy()


@pytest.mark.parametrize("C", [1, 2, 10, 100, 1000])
@pytest.mark.parametrize("prepared", [False, True])
def test_svm_random_within_tolerance(lb, C, prepared):
    desc, W, b = _svm_inputs(200 if prepared else 70, C, seed=C)  # >= 128 -> tensor cores
    s, lab, top = _gpu_svm(lb, desc, W, b, prepared=prepared)
    s_ref, lab_ref, top_ref = oracle.svm_score(desc, W, b)
    ok, worst = svm_tolerance_ok(desc, W, b, s, s_ref)
    assert ok, worst
    assert labels_agree_away_from_ties(s_ref, lab, lab_ref, desc, W, b)
    assert np.array_equal(top, s[np.arange(len(lab)), np.where(lab < 0, 0, lab)])


@pytest.mark.parametrize("prepared", [False, True])
def test_svm_integer_weights_bitexact(lb, prepared):
    """Integer W, b: exact in any summation order -> bit-exact scores and labels."""
    desc, _, _ = _svm_inputs(40, 1, seed=9)
    rng = np.random.default_rng(1)
    W = rng.integers(-1000, 1001, (100, desc.shape[1])).astype(np.float32)
    b = rng.integers(-50, 51, 100).astype(np.float32)
    s, lab, top = _gpu_svm(lb, desc, W, b, prepared=prepared)
    s_ref, lab_ref, top_ref = oracle.svm_score(desc, W, b)
    assert np.array_equal(s, s_ref) and np.array_equal(lab, lab_ref) and np.array_equal(top, top_ref)


def test_svm_ties_and_reject(lb):
    desc, W, b = _svm_inputs(20, 4, seed=3)
    W[2] = W[1]
    b[2] = b[1] = 1e4  # classes 1 and 2 tie at the top -> label 1
    s, lab, top = _gpu_svm(lb, desc, W, b)
    assert (lab == 1).all()
    _, lab, _ = _gpu_svm(lb, desc, W, b, reject=float("inf"))
    assert (lab == -1).all()
    _, lab_r, _ = _gpu_svm(lb, desc, W, b, reject=float(np.median(top)))
    s_ref, lab_ref, _ = oracle.svm_score(desc, W, b, reject_threshold=float(np.median(top)))
    assert np.array_equal(lab_r, lab_ref)


def test_recognize_host_matches_device_path(lb):
    n = 32
    grey, depth = synthgen.face_crops(n, 128, 128, seed=10)
    rois = synthgen.full_rois(n, 128, 128)
    W, b = synthgen.svm_weights(10, 3776, seed=2)
    g = torch.from_numpy(grey).pin_memory()
    d = torch.from_numpy(depth.view(np.int16)).view(torch.uint16).pin_memory()
    r = torch.from_numpy(rois).pin_memory()
    Wt, bt = torch.from_numpy(W).to(DEV), torch.from_numpy(b).to(DEV)
    geom = lb.images_geometry(g, d)
    ws = torch.empty(lb.lbp_recognize_workspace_bytes(geom, True, n, 8, 8, 59), dtype=torch.uint8,
                     device=DEV)
    lab = torch.empty(n, dtype=torch.int32).pin_memory()
    top = torch.empty(n, dtype=torch.float32).pin_memory()
    lb.lbp_recognize_host(g, d, r, 600, 1400, 8, 8, 59, Wt, bt, None, ws, lab, top)
    torch.cuda.synchronize()
    desc = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 59)
    s_ref, lab_ref, top_ref = oracle.svm_score(desc, W, b)
    assert labels_agree_away_from_ties(s_ref, lab.numpy(), lab_ref, desc, W, b)
    ok, _ = svm_tolerance_ok(desc, W, b, top.numpy()[:, None], top_ref[:, None])
    assert ok


def test_svm_prepare_digit_roundtrip(lb):
    """Workspace digits reconstruct W: |m_c sum_k 2^-(8+9k) q_k - W| <= 2^-36 m_c."""
    C, D = 7, 3776
    W, _ = synthgen.svm_weights(C, D, seed=5)
    W[3] = 0.0
    W[4, 10] = 3.0  # exact power-of-two maximum
    Wt = torch.from_numpy(W).to(DEV)
    ws = lb.svm_prepare(Wt)
    torch.cuda.synchronize()
    raw = ws.cpu().numpy()
    scale_off, q_off = 1024, (1024 + 4 * C + 1023) // 1024 * 1024
    m = raw[scale_off:scale_off + 4 * C].view(np.float32)
    rows = ((4 * C + 16) + 31) // 32 * 32
    dpad = (D + 63) // 64 * 64
    stored = raw[q_off:q_off + rows * dpad * 2].view(np.float16).reshape(rows, dpad)
    # pair-major storage (svm_gemm.cuh): CTA r of the pair holds natural rows
    # hh*nn + r*nn/2 + [0, nn/2) of MMA half hh, its half of the pass stored contiguously
    nh = 2 if rows > 256 else 1
    nn = rows // nh
    q = np.empty((rows, dpad))
    for sr in range(rows):
        cr, within = divmod(sr, rows // 2)
        hh, j = divmod(within, nn // 2)
        q[hh * nn + cr * (nn // 2) + j] = stored[sr]
    for c in range(C):
        assert m[c] >= np.abs(W[c]).max() and np.log2(m[c]) == np.round(np.log2(m[c]))
        rec = m[c] * sum(q[4 * c + k, :D] * 2.0 ** -(8 + 9 * k) for k in range(4))
        assert np.abs(q[4 * c:4 * c + 4]).max() <= 256
        assert np.abs(rec - W[c].astype(np.float64)).max() <= 2.0 ** -36 * m[c]
    assert (q[4 * C, :D] == 1).all() and (q[4 * C, D:] == 0).all()


@pytest.mark.parametrize("C", [130, 250])
def test_svm_gemm_multi_pass(lb, C):
    desc, W, b = _svm_inputs(300, C, seed=C)
    s, lab, top = _gpu_svm(lb, desc, W, b, prepared=True)
    s_ref, lab_ref, _ = oracle.svm_score(desc, W, b)
    ok, worst = svm_tolerance_ok(desc, W, b, s, s_ref)
    assert ok, worst
    assert labels_agree_away_from_ties(s_ref, lab, lab_ref, desc, W, b)


@pytest.mark.parametrize("kind", ["big_count", "inf_bits", "mid_count", "big_sum"])
def test_svm_gemm_exactness_fallback(lb, kind):
    """Tiles breaking the exact-accumulation preconditions take the fp64 fallback; counts in
    [1024, 2048) are still exact on the tensor-core path (fp16 exponent field 1)."""
    rng = np.random.default_rng(3)
    n, D, C = 300, 3776, 20
    if kind in ("big_count", "inf_bits", "mid_count"):
        desc = rng.integers(0, 9, (n, D)).astype(np.uint16)  # row sums ~15k < 2^16
        if kind == "big_count":
            desc[5, 17] = 2048
            desc[290, 3] = 40000
        elif kind == "inf_bits":
            desc[7, 100] = 0x7C00  # +Inf as fp16 bits; 0x7E00 = NaN
            desc[260, 64] = 0x7E00
        else:
            desc[5, 17], desc[150, 3], desc[299, 3775] = 1024, 1500, 2047
    else:
        desc = rng.integers(0, 1000, (n, D)).astype(np.uint16)  # sum_d x_d >> 2^17
    W, b = synthgen.svm_weights(C, D, seed=11)
    s, lab, top = _gpu_svm(lb, desc, W, b, prepared=True)
    s_ref, lab_ref, _ = oracle.svm_score(desc, W, b)
    ok, worst = svm_tolerance_ok(desc, W, b, s, s_ref)
    assert ok, worst


def test_svm_single_crop_config1(lb):
    desc, W, b = _svm_inputs(1, 2, seed=1)
    for prepared in (False, True):
        s, lab, top = _gpu_svm(lb, desc, W, b, prepared=prepared)
        s_ref, lab_ref, _ = oracle.svm_score(desc, W, b)
        assert svm_tolerance_ok(desc, W, b, s, s_ref)[0]
        assert labels_agree_away_from_ties(s_ref, lab, lab_ref, desc, W, b)


@pytest.mark.parametrize("kind", ["few_big", "many_big", "plain"])
def test_svm_gemm_i8_counts_above_255(lb, kind):
    """C > 124 takes the INT8 digit-plane kernel: counts above 255 enter the GEMM as their low
    byte and their high part is added exactly (rows with > 8 such entries: fp64)."""
    rng = np.random.default_rng(11)
    n, D, C = 300, 3776, 150
    desc = rng.integers(0, 9, (n, D)).astype(np.uint16)
    if kind == "few_big":
        for r in range(0, n, 7):
            cols = rng.choice(D, 3, replace=False)
            desc[r, cols] = rng.integers(256, 3000, 3)
        desc[5, 0], desc[6, D - 1] = 256, 65535
    elif kind == "many_big":
        desc[[3, 150, 299], :40] = 300
    W, b = synthgen.svm_weights(C, D, seed=12)
    s, lab, top = _gpu_svm(lb, desc, W, b, prepared=True)
    s_ref, lab_ref, _ = oracle.svm_score(desc, W, b)
    ok, worst = svm_tolerance_ok(desc, W, b, s, s_ref)
    assert ok, worst
    assert labels_agree_away_from_ties(s_ref, lab, lab_ref, desc, W, b)


def test_svm_prepare_i8_digit_roundtrip(lb):
    """INT8 workspace (C > 124): W = m (2 u - 1), u = sum_k d_k 2^-(8(k+1)), |error| <= 2^-40 m."""
    C, D = 130, 640
    W, _ = synthgen.svm_weights(C, D, seed=6)
    W[3] = 0.0
    W[4, 10] = 2.0
    ws = lb.svm_prepare(torch.from_numpy(W).to(DEV))
    torch.cuda.synchronize()
    raw = ws.cpu().numpy()
    scale_off, q_off = 1024, (1024 + 4 * C + 1023) // 1024 * 1024
    m = raw[scale_off:scale_off + 4 * C].view(np.float32).astype(np.float64)
    npass, dpad = -(-C // 96), 640
    q = raw[q_off:q_off + npass * 512 * dpad].reshape(npass, 512, dpad).astype(np.float64)
    nat = np.empty_like(q)
    for sr in range(512):  # pair-major storage -> natural rows (TMEM columns)
        cr, within = divmod(sr, 256)
        nat[:, (within // 128) * 256 + cr * 128 + within % 128] = q[:, sr]
    for c in range(C):
        p, j = divmod(c, 96)
        u = sum(nat[p, k * 96 + j, :D] * 2.0 ** (-8 * (k + 1)) for k in range(5))
        assert m[c] > np.abs(W[c]).max() and np.log2(m[c]) == np.round(np.log2(m[c]))
        assert np.abs(m[c] * (2 * u - 1) - W[c].astype(np.float64)).max() <= 2.0 ** -40 * m[c]
    assert (nat[:, 480, :D] == 1).all() and (nat[:, 480, D:] == 0).all()


@pytest.mark.parametrize("C", [130, 8])
def test_svm_fp16_multi_pass_wide_descriptors(lb, C):
    """dim above the INT8 layout's limit (33,000): the fp16 scorer, in 2 passes for C = 130
    (124 + 6 classes) -- both epilogue warps of each lane quarter on a short last pass -- and
    one short pass for C = 8 (the helper warps have at most one 8-class group)"""
    rng = np.random.default_rng(C)
    n, D = 160, 16 * 16 * 256 * 2 // 2 + 4096  # 36,864 dims
    desc = rng.integers(0, 3, (n, D)).astype(np.uint16)
    W, b = synthgen.svm_weights(C, D, seed=C)
    s, lab, top = _gpu_svm(lb, desc, W, b, prepared=True)
    s_ref, lab_ref, _ = oracle.svm_score(desc, W, b)
    ok, worst = svm_tolerance_ok(desc, W, b, s, s_ref)
    assert ok, worst
    assert labels_agree_away_from_ties(s_ref, lab, lab_ref, desc, W, b)


@pytest.mark.parametrize("C", [100, 1000])  # fp16 and INT8 digit-plane layouts
def test_svm_prepared_for_another_model_is_refused(lb, C):
    """a workspace prepared for another W of the same shape, or for a larger model,
    is detected on the device (header layout + 8 sampled weights): every row gets
    LBP_LABEL_BAD_MODEL and NaN scores, nothing past the header is read.  The right workspace
    still scores within R13; a workspace that is too small is refused by the binding and, on
    the host, by the C ABI (tests/test_abi.py)."""
    desc, W1, b = _svm_inputs(300, C, seed=7)
    W2 = W1.copy()
    W2[C - 1, desc.shape[1] - 1] += 0.25  # differs at a sampled position (the last weight)
    W3, _ = synthgen.svm_weights(C + 40, desc.shape[1], seed=8)
    d = torch.from_numpy(desc.view(np.int16)).to(DEV).view(torch.uint16)
    W1t, W2t, W3t = (torch.from_numpy(x).to(DEV) for x in (W1, W2, W3))
    bt = torch.from_numpy(b).to(DEV)
    prep1 = lb.svm_prepare(W1t)
    s, lab, top = lb.svm_score(d, W2t, bt, prepared=prep1)
    torch.cuda.synchronize()
    assert (lab == lb.lbpfused.LBP_LABEL_BAD_MODEL).all().item()
    assert torch.isnan(top).all().item() and torch.isnan(s).all().item()
    prep3 = lb.svm_prepare(W3t)  # larger: passes the size check, fails the header check
    s, lab, top = lb.svm_score(d, W1t, bt, prepared=prep3)
    torch.cuda.synchronize()
    assert (lab == lb.lbpfused.LBP_LABEL_BAD_MODEL).all().item()
    s, lab, top = lb.svm_score(d, W1t, bt, prepared=prep1)  # the right one
    s_ref, lab_ref, _ = oracle.svm_score(desc, W1, b)
    ok, worst = svm_tolerance_ok(desc, W1, b, s.cpu().numpy(), s_ref)
    assert ok, worst
    with pytest.raises(ValueError):
        lb.svm_score(d, W1t, bt, prepared=prep1[:100])
