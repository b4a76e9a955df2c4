"""Multi-rank host logic on CPU (gloo): sharding arithmetic, rank-independent synthetic crops,
and the database all-gather (config 5) against the oracle's single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synthgen
from paper_1504_01883_b200.parallel import gather_database, gather_database_chunked, shard_range


def test_shard_range_covers_exactly():
    for n in (0, 1, 7, 16, 1000, 1 << 20):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (f0, c0), (f1, _) in zip(spans, spans[1:]):
                assert f0 + c0 == f1
            assert sum(c for _, c in spans) == n
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_crops_independent_of_sharding():
    """Crop i is the same whichever rank draws it (weak-scaling invariant)."""
    g_all, d_all = synthgen.face_crops(12, 64, 64, seed=5)
    for world in (2, 3, 4):
        for r in range(world):
            first, count = shard_range(12, r, world)
            g, d = synthgen.face_crops(count, 64, 64, seed=5, first_index=first)
            assert np.array_equal(g, g_all[first:first + count])
            assert np.array_equal(d, d_all[first:first + count])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_total, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        first, count = shard_range(n_total, rank, world)
        grey, depth = synthgen.face_crops(count, 64, 64, seed=9, first_index=first)
        rois = synthgen.full_rois(count, 64, 64)
        desc = oracle.lbp_extract(grey, depth, rois, 600, 1400, 8, 8, 59)  # stand-in extractor
        labels = (np.arange(first, first + count) % 7).astype(np.int32)
        full, lab = gather_database(torch.from_numpy(desc.view(np.int16)).view(torch.uint16),
                                    torch.from_numpy(labels), n_total)
        np.save(os.path.join(out_dir, f"desc{rank}.npy"), full.view(torch.int16).numpy())
        np.save(os.path.join(out_dir, f"lab{rank}.npy"), lab.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_total", [(2, 10), (3, 11)])
def test_gather_database_gloo(tmp_path, world, n_total):
    mp.spawn(_worker, args=(world, _free_port(), n_total, str(tmp_path)), nprocs=world, join=True)
    grey, depth = synthgen.face_crops(n_total, 64, 64, seed=9)
    ref = oracle.lbp_extract(grey, depth, synthgen.full_rois(n_total, 64, 64), 600, 1400, 8, 8, 59)
    for r in range(world):
        got = np.load(tmp_path / f"desc{r}.npy").view(np.uint16)
        lab = np.load(tmp_path / f"lab{r}.npy")
        assert np.array_equal(got, ref)
        assert np.array_equal(lab, np.arange(n_total) % 7)


def _worker_chunked(rank, world, port, n_total, chunks, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        first, count = shard_range(n_total, rank, world)
        grey, depth = synthgen.face_crops(count, 32, 32, seed=9, first_index=first)

        def extract_chunk(lo, hi):  # stand-in extractor on CPU: the oracle
            d = oracle.lbp_extract(grey[lo:hi], depth[lo:hi], synthgen.full_rois(hi - lo, 32, 32),
                                   600, 1400, 4, 4, 59)
            return torch.from_numpy(d.view(np.int16)).view(torch.uint16)
        labels = torch.from_numpy((np.arange(first, first + count) % 5).astype(np.int32))
        full, lab = gather_database_chunked(extract_chunk, labels, n_total, 4 * 4 * 59, chunks,
                                            device=torch.device("cpu"))
        np.save(os.path.join(out_dir, f"desc{rank}.npy"), full.view(torch.int16).numpy())
        np.save(os.path.join(out_dir, f"lab{rank}.npy"), lab.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_total,chunks", [(2, 10, 3), (3, 11, 4), (2, 7, 1), (3, 5, 6)])
def test_gather_database_chunked_gloo(tmp_path, world, n_total, chunks):
    """Overlapped (chunked) database build == the serial one == the oracle, uneven shards and
    more chunks than rows included."""
    mp.spawn(_worker_chunked, args=(world, _free_port(), n_total, chunks, str(tmp_path)),
             nprocs=world, join=True)
    grey, depth = synthgen.face_crops(n_total, 32, 32, seed=9)
    ref = oracle.lbp_extract(grey, depth, synthgen.full_rois(n_total, 32, 32), 600, 1400, 4, 4, 59)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"desc{r}.npy").view(np.uint16), ref)
        assert np.array_equal(np.load(tmp_path / f"lab{r}.npy"), np.arange(n_total) % 5)


# ---- compacted database all-gather (R21) with CPU stand-ins for the
# CUDA pack/unpack that follow the same contract (the oracle's encoding)
def _cpu_pack(desc, row_base, cap, packed_out):
    packed, exc, cnt = oracle.desc_pack_u8(desc.view(torch.int16).numpy().view(np.uint16),
                                           row_base=row_base, cap=cap)
    packed_out[:desc.shape[0]] = torch.from_numpy(packed)
    rec = np.zeros((cap, 4), np.int32)
    if len(exc):
        rec[:len(exc), 0:2] = exc[:, 0].astype(np.int64).view(np.int32).reshape(-1, 2)
        rec[:len(exc), 2] = exc[:, 1]
        rec[:len(exc), 3] = exc[:, 2]
    return torch.from_numpy(rec), torch.tensor([cnt], dtype=torch.int32)


def _cpu_unpack(packed, exc, counts, cap):
    rec = exc.numpy().reshape(-1, cap, 4)
    lists = []
    for l, c in enumerate(counts.tolist()):
        r = rec[l, :min(c, cap)]
        rows = np.ascontiguousarray(r[:, 0:2]).view(np.int64).reshape(-1)
        lists.append(np.stack([rows, r[:, 2].astype(np.int64), r[:, 3].astype(np.int64)], 1))
    out = oracle.desc_unpack_u8(packed.numpy(), np.concatenate(lists) if lists else
                                np.zeros((0, 3), np.int64))
    return torch.from_numpy(out.view(np.int16)).view(torch.uint16)


def _compact_crops(first, count):
    """128x128 crops without depth; every third crop constant (its 36 16x16 cells count 256)"""
    grey, _ = synthgen.face_crops(count, 128, 128, seed=11, first_index=first)
    for k in range(count):
        if (first + k) % 3 == 0:
            grey[k] = 90
    return grey


def _worker_compact(rank, world, port, n_total, cap, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1504_01883_b200.parallel import gather_database_compact
        first, count = shard_range(n_total, rank, world)
        desc = oracle.lbp_extract(_compact_crops(first, count), None,
                                  synthgen.full_rois(count, 128, 128), 0, 0, 8, 8, 59)
        labels = torch.from_numpy((np.arange(first, first + count) % 4).astype(np.int32))
        full, lab = gather_database_compact(torch.from_numpy(desc.view(np.int16)).view(torch.uint16),
                                            labels, n_total, cap=cap, pack=_cpu_pack,
                                            unpack=_cpu_unpack)
        np.save(os.path.join(out_dir, f"desc{rank}.npy"), full.view(torch.int16).numpy())
        np.save(os.path.join(out_dir, f"lab{rank}.npy"), lab.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_total,cap", [(2, 6, 4096), (3, 7, 8), (2, 5, 1)])
def test_gather_database_compact_gloo(tmp_path, world, n_total, cap):
    """u8 + exceptions all-gather == the oracle's u16 matrix; small caps take the re-pack."""
    mp.spawn(_worker_compact, args=(world, _free_port(), n_total, cap, str(tmp_path)),
             nprocs=world, join=True)
    ref = oracle.lbp_extract(_compact_crops(0, n_total), None,
                             synthgen.full_rois(n_total, 128, 128), 0, 0, 8, 8, 59)
    assert (ref > 255).sum() == 36 * len(range(0, n_total, 3))
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"desc{r}.npy").view(np.uint16), ref)
        assert np.array_equal(np.load(tmp_path / f"lab{r}.npy"), np.arange(n_total) % 4)


# ---- fused database build (SURVEY §8e way 2): the host plan, checked by emulating the
# kernel's stores (every ROI row to every destination at the planned offsets) in numpy
def test_fused_gather_layout():
    from paper_1504_01883_b200.parallel import fused_gather_layout
    lay = fused_gather_layout(10, 3776)
    assert lay["pitch"] == 3776 and lay["labels_offset"] == 10 * 3776 * 2
    lay = fused_gather_layout(3, 59)
    assert lay["pitch"] == 64 and lay["labels_offset"] % 16 == 0
    assert lay["bytes"] == lay["labels_offset"] + 12
    with pytest.raises(ValueError):
        fused_gather_layout(3, 0)


@pytest.mark.parametrize("world,n_total,dim,multicast", [(2, 11, 236, False), (3, 10, 59, False),
                                                        (4, 9, 3776, True), (1, 5, 944, False)])
def test_fused_gather_plan_emulated(world, n_total, dim, multicast):
    """Every rank's plan, applied as the kernel applies it, yields the full database in every
    rank's buffer (uneven shards, padded pitch, multicast = one address for all)."""
    from paper_1504_01883_b200 import lbpfused
    from paper_1504_01883_b200.parallel import fused_gather_plan
    rng = np.random.default_rng(world * 100 + n_total)
    db = rng.integers(0, 300, (n_total, dim)).astype(np.uint16)
    labels = rng.integers(0, 50, n_total).astype(np.int32)
    plans = [fused_gather_plan(n_total, r, world, dim, 0xABC0 if multicast else 0,
                               [0x1000 * (r2 + 1) for r2 in range(world)]) for r in range(world)]
    size = plans[0]["bytes"]
    bufs = {0x1000 * (r + 1): np.full(size, 0xEE, np.uint8) for r in range(world)}
    for r, p in enumerate(plans):
        assert p["mode"] == (lbpfused.LBP_GATHER_MULTIMEM if multicast else lbpfused.LBP_GATHER_PEERS)
        targets = list(bufs) if multicast else p["bases"]  # multicast reaches every rank
        for n in range(p["count"]):
            row = np.zeros(p["pitch"], np.uint16)
            row[:dim] = db[p["row_base"] + n]
            off = p["desc_offset"] + (p["row_base"] + n) * p["pitch"] * 2
            lab_off = p["labels_offset"] + 4 * (p["row_base"] + n)
            for t in targets:
                bufs[t][off:off + 2 * p["pitch"]] = row.view(np.uint8)
                bufs[t][lab_off:lab_off + 4] = labels[p["row_base"] + n:p["row_base"] + n + 1].view(np.uint8)
    assert sum(p["count"] for p in plans) == n_total
    for b in bufs.values():
        rows = b[:n_total * plans[0]["pitch"] * 2].view(np.uint16).reshape(n_total, -1)
        assert np.array_equal(rows[:, :dim], db) and not rows[:, dim:].any()
        lab_off = plans[0]["labels_offset"]
        assert np.array_equal(b[lab_off:lab_off + 4 * n_total].view(np.int32), labels)
