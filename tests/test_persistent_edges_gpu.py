"""Batch sizes at the edges of the persistent TMA kernels' scheduling (crop position i of CTA b
is crop b + i * grid; groups take positions i, i + 3, ...; the stage of position i is refilled
with position i + 3 by whichever half-group releases it second): batches of exactly one
position for some CTAs and none for others, one or two positions per group, the first
positions that wrap the stage ring -- for every output mode of the lane kernel (u16, u8
compact, fused grey||depth, depth source) and the tile kernel (64 / 100 / 200 px), bit-exact
against the oracle."""
import numpy as np
import pytest
import torch

import oracle
import synthgen

pytestmark = pytest.mark.gpu

DEV = "cuda"
SIZES = [148, 149, 150, 296, 297, 443, 444, 445, 889]


@pytest.fixture(scope="module")
def lb():
    import paper_1504_01883_b200 as lb
    lb.lbpfused.lib()
    return lb


def _dev(grey, depth, pitch=None):
    g = torch.from_numpy(np.ascontiguousarray(grey)).to(DEV)
    d = torch.from_numpy(np.ascontiguousarray(depth).view(np.int16)).to(DEV)
    if pitch is not None:
        gb = torch.zeros((*g.shape[:2], pitch), dtype=g.dtype, device=DEV)
        gb[:, :, :g.shape[2]] = g
        g = gb[:, :, :g.shape[2]]
        db = torch.zeros((*d.shape[:2], pitch), dtype=d.dtype, device=DEV)
        db[:, :, :d.shape[2]] = d
        d = db[:, :, :d.shape[2]]
    return g, d.view(torch.uint16)


@pytest.mark.parametrize("n", SIZES)
def test_lane59_modes_at_schedule_edges(lb, n):
    grey, depth = synthgen.face_crops(n, 128, 128, seed=n)
    rois = synthgen.full_rois(n, 128, 128)
    g, d = _dev(grey, depth)
    r = torch.from_numpy(rois).to(DEV)
    u16 = lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59)
    cd = lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59)
    fused = lb.lbp_extract_source(g, d, r, 600, 1400, 8, 8, 59, lb.LBP_SRC_FUSED)
    dsrc = lb.lbp_extract_source(None, d, r, 600, 1400, 8, 8, 59, lb.LBP_SRC_DEPTH)
    torch.cuda.synchronize()
    ref = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 59)
    ref_f = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 59, source=2)
    ref_d = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 59, source=1)
    as_u16 = lambda t: t.cpu().view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(as_u16(u16), ref)
    assert np.array_equal(as_u16(fused), ref_f)
    assert np.array_equal(as_u16(dsrc), ref_d)
    assert np.array_equal(cd.packed.cpu().numpy()[:, :ref.shape[1]], (ref & 255).astype(np.uint8))
    assert np.array_equal(cd.exc_n.cpu().numpy(), (ref > 255).sum(1))


@pytest.mark.parametrize("T,pitch", [(64, None), (100, 112), (200, 208)])
@pytest.mark.parametrize("n", [148, 149, 297, 445])
def test_tile_at_schedule_edges(lb, T, pitch, n):
    grey, depth = synthgen.face_crops(n, T, T, seed=T * n)
    rois = synthgen.full_rois(n, T, T)
    g, d = _dev(grey, depth, pitch)
    out = lb.lbp_fused_extract(g, d, torch.from_numpy(rois).to(DEV), 600, 1400, 8, 8, 59)
    torch.cuda.synchronize()
    ref = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 59)
    assert np.array_equal(out.cpu().view(torch.int16).numpy().view(np.uint16), ref)
