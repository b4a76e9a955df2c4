"""GPU parity of the tile variant of the TMA extraction kernel (csrc/lbp_hist_tile.cuh):
crop stacks of 64x64 (two crops per warp row) and 200x200 (the paper's resized face, P:154;
four quadrant tiles per crop) ROIs, 8x8 cells, 59 bins, against the CPU oracle, bit-exact.

Batches of >= 148 ROIs take the tile kernel (smaller ones the band kernel); odd counts leave
the last 64-px pair half empty; ROIs that are not full T x T crops take the generic code
path inside the same kernel, per tile; the depth window exercises the three mask modes
(centred fp16 |d - mid| <= half, two fp16 compares, integer compares) and no depth plane."""
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


def _padded(t, pitch):
    """[n][H][W] CUDA tensor -> a view of a [n][H][pitch] buffer (rows `pitch` elements apart)."""
    if pitch is None or pitch == t.shape[2]:
        return t
    buf = torch.zeros((t.shape[0], t.shape[1], pitch), dtype=t.dtype, device=t.device)
    buf[:, :, :t.shape[2]] = t
    return buf[:, :, :t.shape[2]]


def _extract(lb, grey, depth, rois, dmin, dmax, pitch=None):
    g = _padded(torch.from_numpy(np.ascontiguousarray(grey)).to(DEV), pitch)
    d = None if depth is None else torch.from_numpy(
        np.ascontiguousarray(depth).view(np.int16)).to(DEV)
    d = None if d is None else _padded(d, pitch).view(torch.uint16)
    r = torch.from_numpy(np.ascontiguousarray(rois, dtype=np.int32)).to(DEV)
    st = torch.full((r.shape[0],), 123, dtype=torch.int32, device=DEV)
    out = lb.lbp_fused_extract(g, d, r, dmin, dmax, 8, 8, 59, roi_status=st)
    torch.cuda.synchronize()
    return out.cpu().view(torch.int16).numpy().view(np.uint16), st.cpu().numpy()


def _check(lb, grey, depth, rois, dmin=600, dmax=1400, pitch=None):
    got, st = _extract(lb, grey, depth, rois, dmin, dmax, pitch)
    ref, st_ref = oracle.lbp_extract(grey, depth, rois, dmin, dmax, 8, 8, 59, return_status=True)
    assert np.array_equal(st, st_ref)
    bad = np.nonzero((got != ref).any(1))[0]
    assert bad.size == 0, f"{bad.size} rows differ, first {bad[:5]}"


# 200-px rows need a 16-B multiple pitch for TMA (208 B grey; depth rows are 400 B): the tight
# pitch takes the band kernel, also checked here
@pytest.mark.parametrize("T,n,pitch", [(64, 301, None), (64, 300, None), (200, 160, 208),
                                       (200, 161, 224), (200, 160, None), (100, 150, 112),
                                       (100, 151, None)])
@pytest.mark.parametrize("dist", ["face", "noise", "constant"])
def test_tile_crops_bitexact(lb, T, n, pitch, dist):
    grey, depth = synthgen.face_crops(n, T, T, seed=T + n, dist=dist)
    _check(lb, grey, depth, synthgen.full_rois(n, T, T), pitch=pitch)


@pytest.mark.parametrize("T", [64, 100, 200])
@pytest.mark.parametrize("window", [(600, 1400), (500, 3000), (0, 40000), (0, 0), None])
def test_tile_window_modes(lb, T, window):
    n = 160 if T >= 100 else 297
    pitch = {64: None, 100: 112, 200: 208}[T]
    grey, depth = synthgen.face_crops(n, T, T, seed=7 * T, dist="face")
    if window is None:
        _check(lb, grey, None, synthgen.full_rois(n, T, T), pitch=pitch)
    else:
        _check(lb, grey, depth, synthgen.full_rois(n, T, T), *window, pitch=pitch)


@pytest.mark.parametrize("T", [64, 100, 200])
def test_tile_mixed_rois(lb, T):
    """Full crops mixed with ROIs the tile path does not take (smaller, offset, clamped,
    out-of-range image, too small for the grid): those go through the generic code path
    inside the same kernel; statuses and rows must still match the oracle."""
    n = 170 if T >= 100 else 311
    grey, depth = synthgen.face_crops(n, T, T, seed=99 + T)
    rois = synthgen.full_rois(n, T, T)
    rng = np.random.default_rng(T)
    for i in rng.choice(n, size=n // 5, replace=False):
        kind = i % 5
        if kind == 0:
            rois[i, 1:] = (3, 5, T - 10, T - 7)        # inside, not a full crop
        elif kind == 1:
            rois[i, 1:] = (T // 2, T // 3, T, T)        # clamped at the image edge
        elif kind == 2:
            rois[i, 0] = n + 3                          # no such image: LBP_E_ROI
        elif kind == 3:
            rois[i, 1:] = (0, 0, 6, 6)                  # fewer interior pixels than cells
        else:
            rois[i, 1:] = (16, 0, T - 16, T)            # aligned x, narrower
    _check(lb, grey, depth, rois, pitch={64: None, 100: 112, 200: 208}[T])


@pytest.mark.parametrize("T", [64, 100, 200])
def test_tile_full_size_sample(lb, T):
    """16,384 crops of 64x64 / 200x200 (the bench's tile workloads, 200-px grey rows padded to
    208 B as there): rows of a seeded sample of crops against the oracle computed on those
    crops only."""
    n = 16384
    dev = torch.device(DEV)
    g, d = synthgen.gpu_face_crops(n, T, T, seed=5, device=dev)
    g = _padded(g, {64: None, 100: 112, 200: 208}[T])
    d = _padded(d.view(torch.int16), 112 if T == 100 else None).view(torch.uint16)
    r = torch.from_numpy(synthgen.full_rois(n, T, T)).to(dev)
    out = lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59)
    torch.cuda.synchronize()
    idx = np.sort(np.random.default_rng(1).choice(n, size=48, replace=False))
    ti = torch.as_tensor(idx, device=dev)
    grey = np.ascontiguousarray(g[ti].cpu().numpy())
    depth = d.view(torch.int16)[ti].cpu().numpy().view(np.uint16)
    ref = oracle.lbp_extract(grey, depth, synthgen.full_rois(idx.size, T, T), 600, 1400, 8, 8, 59)
    got = out.view(torch.int16)[ti].cpu().numpy().view(np.uint16)
    assert np.array_equal(got, ref)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("geom", ["frame256_roi100", "tile200_mixed", "tile64_mixed",
                                  "tile100_mixed", "crops128_bins256_mixed"])
def test_generic_positions_repeat_no_hang(lb, geom):
    """Large batches whose ROIs take the generic code path inside the persistent TMA kernels,
    launched repeatedly: a generic position releases its (unfilled) stage with a plain
    mbarrier arrive, which must wait until every thread of the group has passed its wait on
    the current phase (an earlier arrive completes the next phase at once and a late thread
    then waits on the phase after it: a deadlock that showed up within a few launches).
    Rows of a sample are checked against the oracle on every launch."""
    dev = torch.device(DEV)
    if geom == "frame256_roi100":
        n, T, S = 2048, 100, 256     # lane59 FRAME variant, every ROI generic
    elif geom == "tile200_mixed":
        n, T, S = 2048, 200, 200     # tile kernel, quadrants + generic crops
    elif geom == "tile64_mixed":
        n, T, S = 4096, 64, 64       # tile kernel, crop pairs + generic crops
    elif geom == "tile100_mixed":
        n, T, S = 2048, 100, 100     # tile kernel, two stages per group + generic crops
    else:
        n, T, S = 2048, 128, 128     # lane256 kernel (256 bins) + generic crops
    bins = 256 if geom == "crops128_bins256_mixed" else 59
    g, d = synthgen.gpu_face_crops(n, S, S, seed=3, device=dev)
    if S % 16:
        gb = torch.zeros((n, S, (S + 15) // 16 * 16), dtype=torch.uint8, device=dev)
        gb[:, :, :S] = g
        g = gb[:, :, :S]
    if (2 * S) % 16:  # depth rows to a 16-B multiple too (100 px: 200 -> 208 B)
        db = torch.zeros((n, S, (S + 7) // 8 * 8), dtype=torch.int16, device=dev)
        db[:, :, :S] = d.view(torch.int16)
        d = db[:, :, :S].view(torch.uint16)
    rois = synthgen.full_rois(n, S, S)
    if geom == "frame256_roi100":
        rois[:, 1:] = (37, 45, T, T)
    else:
        rois[::7, 1:] = (3, 2, S - 9, S - 5)   # every 7th crop generic
    r = torch.from_numpy(rois).to(dev)
    idx = np.arange(0, n, n // 24)
    ti = torch.as_tensor(idx, device=dev)
    ref = oracle.lbp_extract(g[ti].cpu().numpy(), d.view(torch.int16)[ti].cpu().numpy().view(np.uint16),
                             np.concatenate([np.arange(idx.size)[:, None], rois[idx, 1:]], 1).astype(np.int32),
                             600, 1400, 8, 8, bins)
    out = torch.empty((n, 64 * bins), dtype=torch.uint16, device=dev)
    for _ in range(40):
        lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, bins, out=out)
        torch.cuda.synchronize()
        assert np.array_equal(out.view(torch.int16)[ti].cpu().numpy().view(np.uint16), ref)


@pytest.mark.parametrize("T", [64, 100, 200])
def test_tile_fused_source_and_compact(lb, T):
    """The tile kernel inside the other entry points: the grey block of the fused grey||depth
    descriptor (row stride 2 dim; the depth block takes the band kernel) and the compact u8
    form (extraction into a scratch, then the row pack) -- both against the oracle."""
    n = 160 if T >= 100 else 301
    grey, depth = synthgen.face_crops(n, T, T, seed=13 * T)
    rois = synthgen.full_rois(n, T, T)
    pitch = {64: None, 100: 112, 200: 208}[T]
    g = _padded(torch.from_numpy(grey).to(DEV), pitch)
    d = _padded(torch.from_numpy(depth.view(np.int16)).to(DEV),
                112 if T == 100 else None).view(torch.uint16)
    r = torch.from_numpy(rois).to(DEV)
    fused = lb.lbp_extract_source(g, d, r, 600, 1400, 8, 8, 59, lb.LBP_SRC_FUSED)
    cd = lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59)
    torch.cuda.synchronize()
    ref_g = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 59)
    ref_f = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 59, source=2)
    got_f = fused.cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got_f, ref_f)
    assert np.array_equal(got_f[:, :ref_g.shape[1]], ref_g)
    packed = cd.packed.cpu().numpy()
    assert np.array_equal(packed[:, :ref_g.shape[1]], (ref_g & 255).astype(np.uint8))
    assert np.array_equal(cd.exc_n.cpu().numpy(), (ref_g > 255).sum(1))
