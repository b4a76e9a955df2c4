"""SURVEY §8a row a8 / §8e on the device: the database build ("online database
generation") with descriptors produced by the CUDA extractor on every rank and moved
between ranks by the all-gather, checked row by row against the oracle.

Two processes share the one GPU of the test box over gloo (nothing in this path waits on
another rank's kernels -- gloo's collectives copy through the host -- so sharing a device is
safe; B200_PROFILING.md).  Every variant of parallel.py runs on CUDA tensors:
gather_database (serial), gather_database_chunked (chunk k's all-gather on a second stream
overlapping chunk k+1's extraction) and gather_database_compact (the CUDA u8 + exception-list
pack / unpack kernels).  Shards are uneven (n_total odd) and large enough for the persistent
TMA kernel (>= 148 crops per rank); every third crop of the compact case is constant so its
16x16 cells count 256 (exceptions)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synthgen

N_TOTAL = 301
H = W = 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _crops(first, count, constant_every=0):
    grey, depth = synthgen.face_crops(count, H, W, seed=13, first_index=first)
    if constant_every:
        for k in range(count):
            if (first + k) % constant_every == 0:
                grey[k] = 77
                depth[k] = 1000  # every pixel inside the window: 16x16 cells count 256
    return grey, depth


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1504_01883_b200 as lb
        from paper_1504_01883_b200.parallel import (gather_database, gather_database_chunked,
                                                    gather_database_compact, shard_range)
        dev = torch.device("cuda", 0)
        first, count = shard_range(N_TOTAL, rank, world)
        labels = (torch.arange(first, first + count, device=dev) % 7).to(torch.int32)
        for variant in ("serial", "chunked", "compact"):
            g, d = _crops(first, count, constant_every=3 if variant == "compact" else 0)
            grey = torch.from_numpy(g).to(dev)
            depth = torch.from_numpy(d.view(np.int16)).to(dev).view(torch.uint16)
            rois = torch.from_numpy(synthgen.full_rois(count, H, W)).to(dev)
            if variant == "chunked":
                desc = torch.empty((count, 3776), dtype=torch.uint16, device=dev)

                def extract_chunk(lo, hi):
                    lb.lbp_fused_extract(grey, depth, rois[lo:hi], 600, 1400, 8, 8, 59,
                                         out=desc[lo:hi])
                    return desc[lo:hi]
                full, lab = gather_database_chunked(extract_chunk, labels, N_TOTAL, 3776, 3,
                                                    device=dev)
            else:
                desc = lb.lbp_fused_extract(grey, depth, rois, 600, 1400, 8, 8, 59)
                if variant == "serial":
                    full, lab = gather_database(desc, labels, N_TOTAL)
                else:
                    full, lab = gather_database_compact(desc, labels, N_TOTAL, cap=16)
            torch.cuda.synchronize()
            assert full.is_cuda and lab.is_cuda
            np.save(os.path.join(out_dir, f"{variant}_desc{rank}.npy"),
                    full.cpu().view(torch.int16).numpy())
            np.save(os.path.join(out_dir, f"{variant}_lab{rank}.npy"), lab.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_database_build_two_ranks_cuda_extractor(tmp_path):
    world = 2
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, str(tmp_path)))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    rois = synthgen.full_rois(N_TOTAL, H, W)
    for variant in ("serial", "chunked", "compact"):
        g, d = _crops(0, N_TOTAL, constant_every=3 if variant == "compact" else 0)
        ref = oracle.lbp_extract(g, d, rois, 600, 1400, 8, 8, 59)
        if variant == "compact":  # the exceptions path is exercised: counts of 256 exist
            assert (ref > 255).sum() > 0
        for r in range(world):
            got = np.load(tmp_path / f"{variant}_desc{r}.npy").view(np.uint16)
            assert got.shape == ref.shape
            bad = np.nonzero((got != ref).any(1))[0]
            assert bad.size == 0, f"{variant} rank {r}: rows {bad[:10]} differ from the oracle"
            assert np.array_equal(np.load(tmp_path / f"{variant}_lab{r}.npy"),
                                  np.arange(N_TOTAL) % 7)
