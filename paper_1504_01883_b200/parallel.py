"""Multi-GPU plumbing of the hot path: crop sharding and the database build.

Crops are independent units, so recognition shards them across ranks with no data-path
collective (weak scaling).  The only exchange step of the method is the online database
build (BASELINE configs[4]): every rank extracts the descriptors of its shard
and an all-gather (NCCL over NVLink on GPUs, gloo on CPU tests) assembles the full
[N][dim] training matrix plus labels on every rank, in global crop order.

Only `torch.distributed` plumbing lives here; the descriptors themselves come from the CUDA
library (`lbpfused.lbp_fused_extract`).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced shard of [0, n_total) for `rank`: (first index, count).

    The first n_total % world ranks get one extra crop, so shards differ by at most 1 and
    rank-major order equals global crop order."""
    if world < 1 or not 0 <= rank < world or n_total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n_total, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, count


def gather_database(local_desc: torch.Tensor, local_labels: torch.Tensor, n_total: int,
                    group=None) -> tuple[torch.Tensor, torch.Tensor]:
    """All-gather the per-rank descriptor shards (u16 [count][dim]) and int32 labels into the
    full matrix [n_total][dim] / labels [n_total] on every rank, in global crop order.

    Shards are padded to the largest shard size for the collective (all_gather_into_tensor
    needs equal sizes) and the padding is dropped afterwards.  u16 rows travel as raw bytes
    (uint8, supported by both NCCL and gloo)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    first, count = shard_range(n_total, rank, world)
    if local_desc.shape[0] != count or local_labels.shape[0] != count:
        raise ValueError(f"rank {rank}: shard has {local_desc.shape[0]} rows, expected {count}")
    if world == 1:
        return local_desc, local_labels
    dim = local_desc.shape[1]
    cap = -(-n_total // world)  # largest shard
    dev = local_desc.device
    send = torch.zeros((cap, 2 * dim), dtype=torch.uint8, device=dev)
    send[:count] = local_desc.contiguous().view(torch.uint8)
    send_lab = torch.full((cap,), -1, dtype=torch.int32, device=dev)
    send_lab[:count] = local_labels
    recv = torch.empty((world * cap, 2 * dim), dtype=torch.uint8, device=dev)
    recv_lab = torch.empty((world * cap,), dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    dist.all_gather_into_tensor(recv_lab, send_lab, group=group)
    if n_total % world == 0:  # equal shards: already contiguous in global order
        return recv.view(torch.uint16), recv_lab
    keep = torch.cat([torch.arange(r * cap, r * cap + shard_range(n_total, r, world)[1])
                      for r in range(world)]).to(dev)
    return recv.index_select(0, keep).view(torch.uint16), recv_lab.index_select(0, keep)


def _gpu_pack(desc, row_base, cap, packed_out):
    from . import lbpfused
    _, exc, count = lbpfused.desc_pack_u8(desc, row_base=row_base, cap=cap,
                                          packed=packed_out[:desc.shape[0]])
    return exc, count


def _gpu_unpack(packed, exc, counts, cap):
    from . import lbpfused
    return lbpfused.desc_unpack_u8(packed, exc, counts, cap)


def gather_database_compact(local_desc: torch.Tensor, local_labels: torch.Tensor, n_total: int,
                            group=None, cap: int = 4096, pack=None, unpack=None
                            ) -> tuple[torch.Tensor, torch.Tensor]:
    """gather_database with compacted descriptors (R21): every rank
    sends its rows as u8 counts (min(count, 255), lbp_desc_pack_u8) plus a list of the
    entries > 255, so the all-gather moves half the bytes; the receiver rebuilds the exact
    u16 matrix (lbp_desc_unpack_u8).  Same result as gather_database.

    The exception lists have a fixed capacity per rank for the collective: each rank packs
    with `cap` records, the counts are all-gathered (one host sync per build), and if any
    rank overflowed every rank re-packs with the largest count.  pack / unpack default to the
    CUDA library; CPU (gloo) tests pass stand-ins with the same contract:
      pack(desc u16 [n][dim], row_base, cap, packed_out u8 [>= n][dim]) -> (exc int32 [cap][4],
           count int32 [1]);  unpack(packed u8 [N][dim], exc int32 [L * cap][4],
           counts int32 [L], cap) -> u16 [N][dim]."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    first, count = shard_range(n_total, rank, world)
    if local_desc.shape[0] != count or local_labels.shape[0] != count:
        raise ValueError(f"rank {rank}: shard has {local_desc.shape[0]} rows, expected {count}")
    if world == 1:
        return local_desc, local_labels
    pack = pack or _gpu_pack
    unpack = unpack or _gpu_unpack
    cap = max(1, int(cap))
    dim = local_desc.shape[1]
    rows_cap = -(-n_total // world)
    dev = local_desc.device
    send = torch.zeros((rows_cap, dim), dtype=torch.uint8, device=dev)
    desc = local_desc.contiguous()
    exc, cnt = pack(desc, first, cap, send)
    counts = torch.empty(world, dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(counts, cnt.reshape(1), group=group)
    most = int(counts.max())
    if most > cap:  # some rank's list overflowed: everyone re-packs with the largest count
        cap = most
        exc, cnt = pack(desc, first, cap, send)
    recv = torch.empty((world * rows_cap, dim), dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    exc_all = torch.empty((world * cap, 4), dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(exc_all, exc[:cap].contiguous(), group=group)
    lab_send = torch.full((rows_cap,), -1, dtype=torch.int32, device=dev)
    lab_send[:count] = local_labels
    lab_recv = torch.empty((world * rows_cap,), dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(lab_recv, lab_send, group=group)
    if n_total % world != 0:  # drop the padding rows (exceptions carry global row numbers)
        keep = torch.cat([torch.arange(r * rows_cap, r * rows_cap + shard_range(n_total, r, world)[1])
                          for r in range(world)]).to(dev)
        recv = recv.index_select(0, keep)
        lab_recv = lab_recv.index_select(0, keep)
    return unpack(recv, exc_all, counts, cap), lab_recv


def gather_database_chunked(extract_chunk, local_labels: torch.Tensor, n_total: int, dim: int,
                            chunks: int, group=None, device=None,
                            comm_stream: torch.cuda.Stream | None = None
                            ) -> tuple[torch.Tensor, torch.Tensor]:
    """Overlapped database build (way 1): the local shard is produced in `chunks`
    row chunks; chunk k's all-gather runs on `comm_stream` while chunk k+1 is being extracted
    on the current stream.  The result equals gather_database's (global crop order).

    extract_chunk(lo, hi) -> u16 [hi - lo][dim]: descriptors of local rows [lo, hi), enqueued
    on the current stream (on CPU / gloo it simply returns them).  Every rank uses the same
    chunk row count (ceil of the largest shard / chunks), padding short chunks for the
    collective; the padding is dropped when the chunk is copied into place."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    first, count = shard_range(n_total, rank, world)
    if local_labels.shape[0] != count:
        raise ValueError(f"rank {rank}: {local_labels.shape[0]} labels, expected {count}")
    if world == 1:  # nothing to exchange: the shard is the database
        return extract_chunk(0, count), local_labels
    chunks = max(1, int(chunks))
    cap = -(-n_total // world)
    rpc = max(1, -(-cap // chunks))  # rows per chunk, identical on every rank
    dev = device if device is not None else local_labels.device
    cuda = dev.type == "cuda"
    spans = [shard_range(n_total, r, world) for r in range(world)]
    out = torch.empty((n_total, 2 * dim), dtype=torch.uint8, device=dev)
    if cuda and comm_stream is None:
        comm_stream = torch.cuda.Stream(dev)
    pending = []
    for k in range(chunks):
        lo, hi = min(k * rpc, count), min((k + 1) * rpc, count)
        part = extract_chunk(lo, hi) if hi > lo else None
        if part is not None and hi - lo == rpc and part.is_contiguous():
            send = part.view(torch.uint8)  # full chunk: sent in place
        else:  # short or empty chunk: padded copy
            send = torch.zeros((rpc, 2 * dim), dtype=torch.uint8, device=dev)
            if part is not None:
                send[:hi - lo] = part.contiguous().view(torch.uint8)
        recv = torch.empty((world * rpc, 2 * dim), dtype=torch.uint8, device=dev)
        if cuda:
            ready = torch.cuda.Event()
            ready.record()
            comm_stream.wait_event(ready)
            with torch.cuda.stream(comm_stream):
                send.record_stream(comm_stream)
                recv.record_stream(comm_stream)
                work = dist.all_gather_into_tensor(recv, send, group=group, async_op=True)
        else:
            work = dist.all_gather_into_tensor(recv, send, group=group, async_op=True)
        pending.append((k, recv, work))
        # place the chunks whose collectives were issued earlier (keeps at most 2 in flight)
        while len(pending) > 1:
            _place(pending.pop(0), out, spans, rpc, comm_stream if cuda else None)
    while pending:
        _place(pending.pop(0), out, spans, rpc, comm_stream if cuda else None)
    if cuda:
        torch.cuda.current_stream(dev).wait_stream(comm_stream)
    # labels: one small all-gather (4 B per crop)
    lab_send = torch.full((cap,), -1, dtype=torch.int32, device=dev)
    lab_send[:count] = local_labels
    lab_recv = torch.empty((world * cap,), dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(lab_recv, lab_send, group=group)
    labels = torch.cat([lab_recv[r * cap:r * cap + spans[r][1]] for r in range(world)])
    return out.view(torch.uint16), labels


def _place(item, out, spans, rpc, stream):
    """Copy chunk k of every rank from the gathered buffer to its global rows."""
    k, recv, work = item
    ctx = torch.cuda.stream(stream) if stream is not None else _nullctx()
    with ctx:
        work.wait()
        for r, (first, count) in enumerate(spans):
            lo, hi = min(k * rpc, count), min((k + 1) * rpc, count)
            if hi > lo:
                out[first + lo:first + hi] = recv[r * rpc:r * rpc + (hi - lo)]


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def build_database(grey: torch.Tensor, depth: torch.Tensor | None, rois: torch.Tensor,
                   labels: torch.Tensor, n_total: int, dmin: int, dmax: int, cells_x: int,
                   cells_y: int, bins: int, group=None, stream=None):
    """Config 5 database build on this rank's shard (rois/labels of the shard, on the GPU):
    extract its descriptors with the CUDA library, then all-gather the training matrix."""
    from . import lbpfused
    desc = lbpfused.lbp_fused_extract(grey, depth, rois, dmin, dmax, cells_x, cells_y, bins,
                                      stream=stream)
    return gather_database(desc, labels, n_total, group=group)
