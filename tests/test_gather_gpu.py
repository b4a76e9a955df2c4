"""SURVEY §8e way 2 on the device: the fused database build ("online database generation",
P:154).  lbp_extract_gather writes every descriptor row from the extraction epilogue into every
destination buffer; each destination must end up holding exactly the oracle's rows at the
planned global rows, zero padding past `dim`, the labels, and nothing else touched.

One GPU: PEERS mode with several destination buffers on the same device stands in for the
peer-mapped buffers of several ranks (the stores are the same st.global.v4 to each base; only
the address range differs).  The multicast mode (multimem.st) needs an NVLS multicast object,
which cuMulticastCreate refuses on the single-GPU test pool (tools/probe_multicast.py,
profiles/r02/multicast_probe.json) -- its code path is compiled, not run here.  FusedDatabase
(symmetric memory + barrier) is run at world size 1, where it falls back to PEERS."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synthgen

pytestmark = pytest.mark.gpu
SENT = 0xEE


def _inputs(n, H, W, seed=21):
    dev = torch.device("cuda", 0)
    g, d = synthgen.face_crops(n, H, W, seed=seed)
    grey = torch.from_numpy(g).to(dev)
    depth = torch.from_numpy(d.view(np.int16)).to(dev).view(torch.uint16)
    rois = torch.from_numpy(synthgen.full_rois(n, H, W)).to(dev)
    return g, d, grey, depth, rois


def _run(n, H, W, cells, bins, n_dst, row_base, pad, with_labels=True, seed=21):
    import paper_1504_01883_b200 as lb
    from paper_1504_01883_b200 import lbpfused
    g, d, grey, depth, rois = _inputs(n, H, W, seed)
    dim = lb.lbp_descriptor_dim(cells, cells, bins)
    pitch = -(-dim // 8) * 8 + pad
    n_total = row_base + n + 3
    lab_off = -(-(n_total * pitch * 2) // 16) * 16
    size = lab_off + 4 * n_total
    dev = grey.device
    bufs = [torch.full((size,), SENT, dtype=torch.uint8, device=dev) for _ in range(n_dst)]
    labels = (torch.arange(n, device=dev, dtype=torch.int32) * 7 + 3) if with_labels else None
    dst = lbpfused.gather_dst(lbpfused.LBP_GATHER_PEERS, [b.data_ptr() for b in bufs], 0, pitch,
                              lab_off if with_labels else -1, row_base)
    lb.lbp_extract_gather(grey, depth, rois, 600, 1400, cells, cells, bins, labels, dst)
    torch.cuda.synchronize()
    ref = oracle.lbp_extract(g, d, synthgen.full_rois(n, H, W), 600, 1400, cells, cells, bins)
    for k, b in enumerate(bufs):
        h = b.cpu().numpy()
        rows = h[:n_total * pitch * 2].view(np.uint16).reshape(n_total, pitch)
        mine = rows[row_base:row_base + n]
        bad = np.nonzero((mine[:, :dim] != ref).any(1))[0]
        assert bad.size == 0, f"dst {k}: rows {bad[:10]} differ from the oracle"
        assert not mine[:, dim:].any(), f"dst {k}: padding not zero"
        other = np.concatenate([h[:row_base * pitch * 2], h[(row_base + n) * pitch * 2:lab_off]])
        assert (other == SENT).all(), f"dst {k}: bytes outside this rank's rows written"
        lab = h[lab_off:lab_off + 4 * n_total].view(np.int32)
        if with_labels:
            assert np.array_equal(lab[row_base:row_base + n], np.arange(n) * 7 + 3)
            rest = np.concatenate([h[lab_off:lab_off + 4 * row_base],
                                   h[lab_off + 4 * (row_base + n):]])
            assert (rest == SENT).all()
        else:
            assert (h[lab_off:] == SENT).all()


@pytest.mark.parametrize("n,n_dst,row_base,pad", [(301, 3, 17, 0), (1000, 2, 0, 8),
                                                   (149, 8, 5, 0), (2000, 1, 123, 16)])
def test_gather_fast_path(n, n_dst, row_base, pad):
    """The headline TMA kernel (128x128, 8x8 cells, 59 bins, >= 148 crops) with the gather
    epilogue: 16-B chunks of the staged row to every destination."""
    _run(n, 128, 128, 8, 59, n_dst, row_base, pad)


@pytest.mark.parametrize("n,H,cells,bins,n_dst", [(20, 128, 8, 59, 3), (150, 64, 4, 59, 2),
                                                  (37, 128, 8, 256, 4), (5, 200, 8, 59, 1),
                                                  (1, 128, 1, 256, 2)])
def test_gather_forward_path(n, H, cells, bins, n_dst):
    """Off the fast path (small batch, other geometry / grid / bin count): extraction into the
    scratch, then the forwarding kernel stores every row to every destination."""
    _run(n, H, H, cells, bins, n_dst, row_base=9, pad=0)


def test_gather_without_labels_and_empty():
    import paper_1504_01883_b200 as lb
    from paper_1504_01883_b200 import lbpfused
    _run(300, 128, 128, 8, 59, 2, row_base=0, pad=0, with_labels=False)
    dev = torch.device("cuda", 0)
    buf = torch.full((64,), SENT, dtype=torch.uint8, device=dev)
    grey = torch.zeros((1, 8, 8), dtype=torch.uint8, device=dev)
    rois = torch.zeros((0, 5), dtype=torch.int32, device=dev)
    dst = lbpfused.gather_dst(lbpfused.LBP_GATHER_PEERS, [buf.data_ptr()], 0, 64, -1, 0)
    lb.lbp_extract_gather(grey, None, rois, 600, 1400, 1, 1, 59, None, dst)
    torch.cuda.synchronize()
    assert (buf.cpu().numpy() == SENT).all()


def test_gather_argument_errors():
    import paper_1504_01883_b200 as lb
    from paper_1504_01883_b200 import lbpfused
    _, _, grey, depth, rois = _inputs(4, 128, 128)
    buf = torch.zeros(1 << 20, dtype=torch.uint8, device=grey.device)
    p = buf.data_ptr()
    bad = [lbpfused.gather_dst(0, [p], 0, 3776, -1, 0),             # unknown mode
           lbpfused.gather_dst(lbpfused.LBP_GATHER_MULTIMEM, [p, p], 0, 3776, -1, 0),
           lbpfused.gather_dst(lbpfused.LBP_GATHER_PEERS, [p + 8], 0, 3776, -1, 0),
           lbpfused.gather_dst(lbpfused.LBP_GATHER_PEERS, [p], 8, 3776, -1, 0),
           lbpfused.gather_dst(lbpfused.LBP_GATHER_PEERS, [p], 0, 3770, -1, 0),
           lbpfused.gather_dst(lbpfused.LBP_GATHER_PEERS, [p], 0, 3768, -1, 0),
           lbpfused.gather_dst(lbpfused.LBP_GATHER_PEERS, [p], 0, 3776, 6, 0),
           lbpfused.gather_dst(lbpfused.LBP_GATHER_PEERS, [p], 0, 3776, -1, -1)]
    for dst in bad:
        with pytest.raises(lbpfused.LbpError):
            lb.lbp_extract_gather(grey, depth, rois, 600, 1400, 8, 8, 59, None, dst)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _fused_db_worker(port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_1504_01883_b200.parallel import FusedDatabase
        n = 333
        g, d, grey, depth, rois = _inputs(n, 128, 128, seed=5)
        labels = torch.arange(n, device=grey.device, dtype=torch.int32) % 11
        db = FusedDatabase(n, 3776, grey.device)
        rows, lab = db.build(grey, depth, rois, labels, 600, 1400, 8, 8, 59)
        torch.cuda.synchronize()
        np.save(out + "/rows.npy", rows.cpu().view(torch.int16).numpy())
        np.save(out + "/lab.npy", lab.cpu().numpy())
        with open(out + "/mode.txt", "w") as f:
            f.write(db.mode)
    finally:
        dist.destroy_process_group()


def test_fused_database_world1(tmp_path):
    import torch.multiprocessing as mp
    p = mp.get_context("spawn").Process(target=_fused_db_worker, args=(_free_port(), str(tmp_path)))
    p.start()
    p.join(300)
    assert p.exitcode == 0
    n = 333
    g, d = synthgen.face_crops(n, 128, 128, seed=5)
    ref = oracle.lbp_extract(g, d, synthgen.full_rois(n, 128, 128), 600, 1400, 8, 8, 59)
    assert np.array_equal(np.load(tmp_path / "rows.npy").view(np.uint16), ref)
    assert np.array_equal(np.load(tmp_path / "lab.npy"), np.arange(n) % 11)
    assert (tmp_path / "mode.txt").read_text() in ("peers", "multimem")
