"""GPU parity of lbp_extract_source (depth-source codes and the fused
grey||depth descriptor) against the oracle's source switch, element by element, bit-exact.
Covers the 128x128 batch shape of the headline configs, ragged ROIs (generic path), pitched
640x480 frames with mixed ROIs, the full u16 depth range, errors and the grey-source
equivalence with lbp_fused_extract."""
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


def _run(lb, grey, depth, rois, dmin, dmax, kx, ky, bins, source, grey_none=False):
    g = None if grey_none else torch.from_numpy(np.ascontiguousarray(grey)).to(DEV)
    d = None if depth is None else _dev_u16(depth)
    r = torch.from_numpy(np.ascontiguousarray(rois, dtype=np.int32)).to(DEV)
    st = torch.full((r.shape[0],), 77, dtype=torch.int32, device=DEV)
    out = lb.lbp_extract_source(g, d, r, dmin, dmax, kx, ky, bins, source, roi_status=st)
    torch.cuda.synchronize()
    return out.cpu().view(torch.int16).numpy().view(np.uint16), st.cpu().numpy()


def _check(lb, grey, depth, rois, dmin, dmax, kx, ky, bins, source, grey_none=False):
    got, st = _run(lb, grey, depth, rois, dmin, dmax, kx, ky, bins, source, grey_none)
    ref, st_ref = oracle.lbp_extract(None if grey_none else grey, depth, rois, dmin, dmax, kx, ky,
                                     bins, source=source, return_status=True)
    assert got.shape == ref.shape
    assert np.array_equal(st, st_ref)
    bad = np.nonzero((got != ref).any(1))[0]
    assert bad.size == 0, f"{bad.size} rows differ, first {bad[:5]}"
    return got


@pytest.mark.parametrize("source", [1, 2])
@pytest.mark.parametrize("bins", [59, 256])
def test_crops_128(lb, source, bins):
    # >= 148 ROIs: the persistent TMA kernels (smaller batches take the band kernel)
    grey, depth = synthgen.face_crops(160, 128, 128, seed=31)
    _check(lb, grey, depth, synthgen.full_rois(160, 128, 128), 600, 1400, 8, 8, bins, source)
    _check(lb, grey[:16], depth[:16], synthgen.full_rois(16, 128, 128), 600, 1400, 8, 8, bins,
           source)


def test_depth_source_without_grey(lb):
    grey, depth = synthgen.face_crops(6, 64, 64, seed=32)
    _check(lb, grey, depth, synthgen.full_rois(6, 64, 64), 600, 1400, 8, 8, 59, 1,
           grey_none=True)


@pytest.mark.parametrize("H,W,kx,ky", [(37, 53, 5, 3), (20, 131, 7, 9), (9, 9, 7, 1)])
def test_ragged_rois(lb, H, W, kx, ky):
    grey, depth = synthgen.face_crops(3, H, W, seed=H * W)
    rois = synthgen.random_rois(25, 3, H, W, seed=kx * ky)
    for source in (1, 2):
        _check(lb, grey, depth, rois, 600, 1400, kx, ky, 59, source)


def test_full_u16_range_and_holes(lb):
    """Depth samples over the whole u16 range (incl. values >= 0x7C00 and 0 holes)."""
    rng = np.random.default_rng(9)
    vals = np.array([0, 1, 2047, 2048, 31743, 31744, 31745, 40000, 65534, 65535], np.uint16)
    depth = vals[rng.integers(0, len(vals), (8, 64, 64))]
    grey = rng.integers(0, 256, (8, 64, 64)).astype(np.uint8)
    rois = synthgen.full_rois(8, 64, 64)
    for source in (1, 2):
        _check(lb, grey, depth, rois, 1, 65535, 8, 8, 256, source)
        _check(lb, grey, depth, rois, 0, 40000, 4, 4, 59, source)


def test_pitched_frames_mixed_rois(lb):
    n_frames, H, W = 9, 480, 640  # 153 ROIs: the persistent TMA kernels
    grey, depth = synthgen.face_crops(n_frames, H, W, seed=33)
    rng = np.random.default_rng(8)
    rois = []
    for f in range(n_frames):
        rois += [[f, 0, 0, 128, 128], [f, 16, 32, 128, 128], [f, 3, 5, 128, 128],
                 [f, -20, -20, 128, 128], [f, 50, 60, 100, 90], [f, 10, 10, 2, 128],
                 [f, 700, 0, 128, 128]]
        for _ in range(10):
            rois.append([f, int(rng.integers(0, W - 128)), int(rng.integers(0, H - 128)), 128, 128])
    rois = np.array(rois, np.int32)
    for source in (0, 1, 2):
        _check(lb, grey, depth, rois, 600, 1400, 8, 8, 59, source)


def test_grey_source_equals_fused_extract(lb):
    grey, depth = synthgen.face_crops(10, 128, 128, seed=34)
    rois = synthgen.full_rois(10, 128, 128)
    a, _ = _run(lb, grey, depth, rois, 600, 1400, 8, 8, 59, 0)
    g = torch.from_numpy(grey).to(DEV)
    b = lb.lbp_fused_extract(g, _dev_u16(depth), torch.from_numpy(rois).to(DEV), 600, 1400, 8, 8,
                             59).cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(a, b)
    f, _ = _run(lb, grey, depth, rois, 600, 1400, 8, 8, 59, 2)
    assert np.array_equal(f[:, :3776], a)


def test_errors(lb):
    grey, depth = synthgen.face_crops(1, 32, 32, seed=1)
    r = torch.from_numpy(synthgen.full_rois(1, 32, 32)).to(DEV)
    g = torch.from_numpy(grey).to(DEV)
    with pytest.raises(lb.LbpError):
        lb.lbp_extract_source(g, None, r, 0, 10, 2, 2, 59, lb.LBP_SRC_DEPTH)
    with pytest.raises(lb.LbpError):
        lb.lbp_extract_source(g, _dev_u16(depth), r, 0, 10, 2, 2, 59, 7)


@pytest.mark.parametrize("dmax", [31742, 31743, 65535])
def test_depth_source_128_full_range(lb, dmax):
    """128x128 crops (the TMA depth-source kernel while dmax <= 0x7BFE, the generic kernel
    above) with neighbours over the whole u16 range: the clamp to 0x7BFF must be exact."""
    rng = np.random.default_rng(dmax)
    vals = np.array([0, 1, 900, 901, 2047, 2048, 31741, 31742, 31743, 31744, 40000, 65535],
                    np.uint16)
    depth = vals[rng.integers(0, len(vals), (150, 128, 128))]
    grey = rng.integers(0, 256, (150, 128, 128)).astype(np.uint8)
    rois = synthgen.full_rois(150, 128, 128)
    for source in (1, 2):
        _check(lb, grey, depth, rois, 1, dmax, 8, 8, 59, source)


@pytest.mark.parametrize("dmin,dmax", [(600, 1400), (600, 1401), (1, 31742), (0, 0)])
def test_fused_one_pass_mixed_rois(lb, dmin, dmax):
    """LBP_SRC_FUSED in ONE pass of the TMA kernel (both code planes of one staged tile): the
    centred (600..1400) and plain fp16 windows, an empty window, fast 128x128 crops mixed with
    ROIs off the TMA path (the in-kernel generic path writes both blocks), >= 148 ROIs."""
    n_img = 60
    grey, depth = synthgen.face_crops(n_img, 128, 128, seed=33)
    grey[5] = 99
    depth[5] = 1000  # uniform crop: counts of 256 in both blocks
    rois = np.concatenate([synthgen.full_rois(n_img, 128, 128),
                           synthgen.random_rois(200, n_img, 128, 128, seed=7)]).astype(np.int32)
    _check(lb, grey, depth, rois, dmin, dmax, 8, 8, 59, 2)


def test_fused_one_pass_large_batch(lb):
    n = 2000
    grey, depth = synthgen.face_crops(n, 128, 128, seed=34)
    _check(lb, grey, depth, synthgen.full_rois(n, 128, 128), 600, 1400, 8, 8, 59, 2)
