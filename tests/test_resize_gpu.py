"""GPU parity of lbp_extract_resized (ROI crop + resize fused into the
histogram staging) against the oracle, element by element, bit-exact: the paper's
200x200, up- and down-scaling, clamped / empty ROIs, every code source, 59/256 bins,
pitched Kinect-shaped frames."""
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


def _dev_u16(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(DEV).view(torch.uint16)


def _check(lb, grey, depth, rois, size, dmin, dmax, kx, ky, bins, source=0):
    g = None if grey is None else torch.from_numpy(np.ascontiguousarray(grey)).to(DEV)
    d = None if depth is None else _dev_u16(depth)
    r = torch.from_numpy(np.ascontiguousarray(rois, dtype=np.int32)).to(DEV)
    st = torch.full((r.shape[0],), 55, dtype=torch.int32, device=DEV)
    out = lb.lbp_extract_resized(g, d, r, size, dmin, dmax, kx, ky, bins, source, roi_status=st)
    torch.cuda.synchronize()
    got = out.cpu().view(torch.int16).numpy().view(np.uint16)
    ref, st_ref = oracle.lbp_extract_resized(grey, depth, rois, size, dmin, dmax, kx, ky, bins,
                                             source=source, return_status=True)
    assert np.array_equal(st.cpu().numpy(), st_ref)
    bad = np.nonzero((got != ref).any(1))[0]
    assert bad.size == 0, f"{bad.size} rows differ, first {bad[:5]}"


def _frame_rois(n_frames, H, W, k, seed):
    rng = np.random.default_rng(seed)
    rois = []
    for f in range(n_frames):
        for _ in range(k):
            w = int(rng.integers(40, 260))
            h = int(rng.integers(40, 260))
            rois.append([f, int(rng.integers(-30, W - 20)), int(rng.integers(-30, H - 20)), w, h])
    rois += [[0, W + 5, 0, 50, 50], [n_frames, 0, 0, 50, 50], [0, 10, 10, 1, 1]]
    return np.array(rois, np.int32)


@pytest.mark.parametrize("size", [200, 128, 64])
@pytest.mark.parametrize("source", [0, 1, 2])
def test_frames_resized(lb, size, source):
    n_frames, H, W = 2, 480, 640
    grey, depth = synthgen.face_crops(n_frames, H, W, seed=size + source)
    rois = _frame_rois(n_frames, H, W, 12, seed=size)
    _check(lb, grey, depth, rois, size, 600, 1400, 8, 8, 59, source)


@pytest.mark.parametrize("bins", [59, 256])
def test_grids_and_no_mask(lb, bins):
    grey, depth = synthgen.face_crops(1, 300, 400, seed=7)
    rois = _frame_rois(1, 300, 400, 8, seed=bins)
    _check(lb, grey, None, rois, 150, 0, 0, 7, 5, bins)
    _check(lb, grey, depth, rois, 97, 600, 1400, 3, 11, bins)
    _check(lb, grey, depth, rois, 40, 1, 65535, 20, 2, bins)   # many cells per row: chunks


def test_large_size_row_chunks(lb):
    """size 1000 (staging in row chunks) and the identity resize of a 128x128 ROI."""
    grey, depth = synthgen.face_crops(1, 480, 640, seed=9)
    _check(lb, grey, depth, [[0, 100, 50, 300, 200], [0, 0, 0, 640, 480]], 1000, 600, 1400, 4,
           4, 59, 2)
    rois = np.array([[0, 64, 32, 128, 128]], np.int32)
    g = torch.from_numpy(grey).to(DEV)
    a = lb.lbp_extract_resized(g, _dev_u16(depth), torch.from_numpy(rois).to(DEV), 128, 600,
                               1400, 8, 8, 59)
    b = lb.lbp_fused_extract(g, _dev_u16(depth), torch.from_numpy(rois).to(DEV), 600, 1400, 8,
                             8, 59)
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
