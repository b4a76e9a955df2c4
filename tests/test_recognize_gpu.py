"""GPU parity of lbp_recognize (extraction + SVM in one call; one fused cluster launch for
small batches) against the oracle: descriptors and statuses bit-exact, scores within the
R13 tolerance, labels equal away from ties, reject threshold; large batches take the
two-kernel path and must agree too."""
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


def _dev_u16(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(DEV).view(torch.uint16)


def _run(lb, grey, depth, rois, kx, ky, bins, C, seed, reject=-math.inf, prepared=False):
    dim = kx * ky * bins
    W, b = synthgen.svm_weights(C, dim, seed=seed)
    Wt, bt = torch.from_numpy(W).to(DEV), torch.from_numpy(b).to(DEV)
    st = torch.full((len(rois),), 9, dtype=torch.int32, device=DEV)
    desc, s, lab, top = lb.lbp_recognize(
        torch.from_numpy(grey).to(DEV), None if depth is None else _dev_u16(depth),
        torch.from_numpy(np.asarray(rois, np.int32)).to(DEV), 600, 1400, kx, ky, bins, Wt, bt,
        prepared=lb.svm_prepare(Wt) if prepared else None, reject_threshold=reject,
        want_scores=True, roi_status=st)
    torch.cuda.synchronize()
    ref, st_ref = oracle.lbp_extract(grey, depth, rois, 600, 1400, kx, ky, bins,
                                     return_status=True)
    got = desc.cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(st.cpu().numpy(), st_ref)
    assert np.array_equal(got, ref)
    s_ref, lab_ref, top_ref = oracle.svm_score(ref, W, b, reject_threshold=reject)
    ok, worst = svm_tolerance_ok(ref, W, b, s.cpu().numpy(), s_ref)
    assert ok, worst
    assert labels_agree_away_from_ties(s_ref, lab.cpu().numpy(), lab_ref, ref, W, b)
    return lab.cpu().numpy(), top.cpu().numpy(), top_ref


@pytest.mark.parametrize("C", [1, 2, 10, 100, 1000])
def test_single_crop_and_frame(lb, C):
    grey, depth = synthgen.face_crops(1, 64, 64, seed=C)
    _run(lb, grey, depth, synthgen.full_rois(1, 64, 64), 8, 8, 59, C, seed=C)
    g, d, rois = synthgen.kinect_frames(2, seed=C)
    _run(lb, g, d, rois, 8, 8, 59, C, seed=C + 1)


def test_grids_bins_errors_and_reject(lb):
    g, d, _ = synthgen.kinect_frames(1, seed=5)
    rois = [[0, 10, 20, 128, 128], [0, 600, 400, 128, 128], [0, 700, 0, 50, 50],
            [0, 3, 5, 2, 40], [0, 100, 100, 97, 61]]
    _run(lb, g, d, rois, 4, 6, 256, 7, seed=2)
    _run(lb, g, None, rois, 8, 3, 59, 3, seed=3)
    lab, top, top_ref = _run(lb, g, d, rois, 8, 8, 59, 10, seed=4, reject=0.0)
    assert ((top < 0.0) == (lab == -1)).all()


def test_large_batch_two_kernel_path(lb):
    grey, depth = synthgen.face_crops(200, 128, 128, seed=8)
    _run(lb, grey, depth, synthgen.full_rois(200, 128, 128), 8, 8, 59, 100, seed=8,
         prepared=True)


def test_wide_cell_rows_and_small_images(lb):
    """cells_x * bins above the 4,096 smem counters (the segment is scored from the written
    descriptor instead of the CTA's histogram), more classes than warps (the W prefetch covers
    only the first class of each warp), and 256- vs 512-thread CTAs (image height < / >= 128)"""
    g, d, _ = synthgen.kinect_frames(1, seed=9)
    rois = [[0, 10, 20, 200, 150], [0, 300, 200, 128, 128]]
    _run(lb, g, d, rois, 20, 4, 256, 40, seed=9)   # 20 x 256 = 5,120 entries per cell row
    _run(lb, g, d, rois, 16, 8, 256, 3, seed=10)   # exactly 4,096
    grey, depth = synthgen.face_crops(3, 100, 120, seed=11)
    _run(lb, grey, depth, synthgen.full_rois(3, 100, 120), 8, 8, 59, 25, seed=11)
