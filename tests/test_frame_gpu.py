"""GPU parity of the FRAME variant of the lane-private TMA kernel (lbp_hist_lane59.cuh: 144-px
grey / 136-px depth boxes at the aligned-down column, so 128x128 ROIs at ANY column of a wider
frame take the TMA path) against the oracle, element by element, bit-exact.

Batches of >= 148 ROIs (smaller batches take the band kernel).  Covers every column residue
mod 16, ROIs flush with the right and bottom frame edges (the staged box runs past the frame:
TMA zero-fills, the kernel must not use those bytes), the narrowest frame the variant takes
(144 px), pitched rows, ROIs that fall back to the generic path inside the kernel (clamped,
odd-sized, bad image), and every kernel instance: grey codes with the fp16 depth window, with
the integer window (dmax > 0x7BFE), without depth, depth-source codes, fused grey||depth."""
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


def _pitched(t, pad):
    """the same [n][H][W] values in rows of W + pad elements (a strided view)"""
    n, H, W = t.shape
    big = torch.zeros((n, H, W + pad), dtype=t.dtype, device=t.device)
    big[:, :, :W] = t
    return big[:, :, :W]


def _frame_rois(n_frames, H, W, seed, per_frame=20, extras=True):
    rng = np.random.default_rng(seed)
    rois = []
    for f in range(n_frames):
        for k in range(per_frame):
            x = (int(rng.integers(0, (W - 128) // 16 + 1)) * 16 + k) % (W - 127)  # residues
            rois.append([f, x, int(rng.integers(0, H - 127)), 128, 128])
        rois.append([f, W - 128, H - 128, 128, 128])  # flush with the right/bottom edges
        rois.append([f, W - 129 if W > 128 else 0, 0, 128, 128])
        if extras:  # generic path inside the kernel
            rois += [[f, -9, 4, 128, 128], [f, W - 100, 7, 128, 128], [f, 5, 6, 100, 90],
                     [f, 3, 3, 128, 127]]
    rois.append([n_frames, 0, 0, 128, 128])  # bad image
    return np.array(rois, np.int32)


def _check(lb, grey, depth, rois, dmin, dmax, source, pad=0, grey_none=False):
    g = None if grey_none else torch.from_numpy(np.ascontiguousarray(grey)).to(DEV)
    d = None if depth is None else _dev_u16(depth)
    if pad:
        g = None if g is None else _pitched(g, pad)
        d = None if d is None else _pitched(d, pad)
    r = torch.from_numpy(rois).to(DEV)
    st = torch.full((r.shape[0],), 77, dtype=torch.int32, device=DEV)
    out = lb.lbp_extract_source(g, d, r, dmin, dmax, 8, 8, 59, source, roi_status=st)
    torch.cuda.synchronize()
    got = out.cpu().view(torch.int16).numpy().view(np.uint16)
    ref, st_ref = oracle.lbp_extract(None if grey_none else grey, depth, rois, dmin, dmax, 8, 8,
                                     59, source=source, return_status=True)
    assert np.array_equal(st.cpu().numpy(), st_ref)
    bad = np.nonzero((got != ref).any(1))[0]
    assert bad.size == 0, f"{bad.size} rows differ, first {bad[:5]} rois {rois[bad[:3]]}"


@pytest.mark.parametrize("source", [0, 1, 2])
def test_frames_every_residue(lb, source):
    grey, depth = synthgen.face_crops(8, 480, 640, seed=51)
    _check(lb, grey, depth, _frame_rois(8, 480, 640, 1), 600, 1400, source)


def test_frames_integer_window_and_no_depth(lb):
    grey, depth = synthgen.face_crops(8, 300, 400, seed=52)
    rois = _frame_rois(8, 300, 400, 2)
    _check(lb, grey, depth, rois, 1, 40000, 0)   # dmax > 0x7BFE: integer window
    _check(lb, grey, depth, rois, 500, 65535, 0)
    _check(lb, grey, None, rois, 0, 0, 0)        # no depth: grey codes, every pixel counted
    _check(lb, grey, depth, rois, 0, 0, 0)       # empty window (only d = 0 is in [0, 0])
    _check(lb, grey, depth, rois, 5, 9, 0)       # a window no pixel falls in


def test_narrowest_frame_and_pitch(lb):
    grey, depth = synthgen.face_crops(10, 130, 144, seed=53)
    rois = _frame_rois(10, 130, 144, 3)
    for source in (0, 1, 2):
        _check(lb, grey, depth, rois, 600, 1400, source)
        _check(lb, grey, depth, rois, 600, 1400, source, pad=48)
    _check(lb, grey, depth, rois, 600, 1400, 1, grey_none=True)


def test_kinect_stream_batch(lb):
    """config2's frame stream batched: 40 frames x 4 tracked faces (160 ROIs)."""
    grey, depth, rois = synthgen.kinect_frames(40, 4, seed=54)
    for source in (0, 1, 2):
        _check(lb, grey, depth, rois, 600, 1400, source)


@pytest.mark.parametrize("bins", [59, 256])
def test_small_batch_band_kernel_512(lb, bins):
    """fewer ROIs than SMs on tall frames: the band kernel with 512-thread CTAs"""
    grey, depth = synthgen.face_crops(3, 480, 640, seed=55)
    rois = _frame_rois(3, 480, 640, 5, per_frame=5)
    assert len(rois) * 8 < 2 * 148
    for source in (0, 1, 2):
        g = torch.from_numpy(grey).to(DEV)
        d = _dev_u16(depth)
        out = lb.lbp_extract_source(g, d, torch.from_numpy(rois).to(DEV), 600, 1400, 8, 8, bins,
                                    source)
        torch.cuda.synchronize()
        ref = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, bins, source=source)
        assert np.array_equal(out.cpu().view(torch.int16).numpy().view(np.uint16), ref)
