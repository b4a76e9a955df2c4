"""GPU parity of the 256-bin lane-private TMA kernel (lbp_hist_lane256.cuh; "0-255" bins,
8x8 cells, 128x128 ROIs) against the oracle, bit-exact: every depth-window mode (integer, fp16
compares, centred), no depth, the all-pixels-one-code constant crops (counts of 256 in the
16x16 cells), noise crops (all 256 codes), mixed ROIs that take the generic path inside the
kernel, frames with aligned and unaligned ROIs, pitched rows, descriptor row strides."""
import numpy as np
import pytest
import torch

import oracle
import synthgen

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def lb():
    import paper_1504_01883_b200 as lb
    lb.lbpfused.lib()
    return lb


def _run(lb, grey, depth, rois, lo, hi, pad=0):
    g = torch.from_numpy(np.ascontiguousarray(grey)).to(DEV)
    d = None if depth is None else \
        torch.from_numpy(np.ascontiguousarray(depth).view(np.int16)).to(DEV).view(torch.uint16)
    if pad:
        n, H, W = g.shape
        gb = torch.zeros((n, H, W + pad), dtype=g.dtype, device=DEV)
        gb[:, :, :W] = g
        g = gb[:, :, :W]
        if d is not None:
            db = torch.zeros((n, H, W + pad), dtype=d.dtype, device=DEV)
            db[:, :, :W] = d
            d = db[:, :, :W]
    r = torch.from_numpy(rois).to(DEV)
    st = torch.full((r.shape[0],), 77, dtype=torch.int32, device=DEV)
    out = lb.lbp_fused_extract(g, d, r, lo, hi, 8, 8, 256, roi_status=st)
    torch.cuda.synchronize()
    return out.cpu().view(torch.int16).numpy().view(np.uint16), st.cpu().numpy()


def _check(lb, grey, depth, rois, lo, hi, pad=0):
    got, st = _run(lb, grey, depth, rois, lo, hi, pad)
    ref, st_ref = oracle.lbp_extract(grey, depth, rois, lo, hi, 8, 8, 256, return_status=True)
    assert np.array_equal(st, st_ref)
    bad = np.nonzero((got != ref).any(1))[0]
    assert bad.size == 0, f"[{lo}, {hi}]: {bad.size} rows differ, first {bad[:5]}"


@pytest.mark.parametrize("lo,hi", [(600, 1400), (601, 1400), (600, 3000), (5, 40000), (0, 0)])
def test_crops_every_window_mode(lb, lo, hi):
    grey, depth = synthgen.face_crops(160, 128, 128, seed=71)
    _check(lb, grey, depth, synthgen.full_rois(160, 128, 128), lo, hi)


def test_no_depth_constant_and_noise_crops(lb):
    grey, _ = synthgen.face_crops(160, 128, 128, seed=72)
    grey[::4] = 99                                                     # one code per crop
    grey[1::4] = np.random.default_rng(3).integers(0, 256, grey[1::4].shape)  # all codes
    ref = oracle.lbp_extract(grey, None, synthgen.full_rois(160, 128, 128), 0, 0, 8, 8, 256)
    assert ref.max() == 256
    _check(lb, grey, None, synthgen.full_rois(160, 128, 128), 0, 0)


def test_frames_mixed_rois_and_pitch(lb):
    grey, depth = synthgen.face_crops(8, 200, 320, seed=73)
    rng = np.random.default_rng(74)
    rois = []
    for f in range(8):
        for _ in range(16):
            rois.append([f, 16 * int(rng.integers(0, 12)), int(rng.integers(0, 73)), 128, 128])
        rois += [[f, 5, 9, 128, 128], [f, -4, 0, 128, 128], [f, 30, 20, 100, 64]]
    rois.append([9, 0, 0, 128, 128])  # bad image
    rois = np.array(rois, np.int32)
    _check(lb, grey, depth, rois, 600, 1400)
    _check(lb, grey, depth, rois, 600, 1400, pad=32)


def test_matches_previous_kernel_layout_in_a_strided_block(lb):
    """lbp_extract_source's fused layout writes the 256-bin grey block with row stride 2 dim"""
    grey, depth = synthgen.face_crops(150, 128, 128, seed=75)
    rois = synthgen.full_rois(150, 128, 128)
    g = torch.from_numpy(grey).to(DEV)
    d = torch.from_numpy(depth.view(np.int16)).to(DEV).view(torch.uint16)
    out = lb.lbp_extract_source(g, d, torch.from_numpy(rois).to(DEV), 600, 1400, 8, 8, 256, 2)
    torch.cuda.synchronize()
    ref = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 256, source=2)
    assert np.array_equal(out.cpu().view(torch.int16).numpy().view(np.uint16), ref)
