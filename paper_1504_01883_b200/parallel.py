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


# ---------------------------------------------------------------------------------------------
# Fused database build (SURVEY §8e way 2): the extraction epilogue writes each descriptor row
# ONCE into every rank's copy of the training matrix -- through an NVLS multicast address when
# the platform gives one (multimem.st; the NVSwitch replicates), else as one store per rank
# buffer mapped over NVLink (P2P).  No separate collective: one cross-rank barrier at the end.

def fused_gather_layout(n_total: int, dim: int) -> dict:
    """Byte layout of the gathered matrix inside one symmetric buffer: rows of `pitch` u16
    (dim rounded up to a multiple of 8, so every row starts 16-B aligned), then int32 labels
    at a 16-B aligned offset."""
    if n_total < 0 or dim < 1:
        raise ValueError("bad layout arguments")
    pitch = -(-dim // 8) * 8
    labels_offset = -(-(n_total * pitch * 2) // 16) * 16
    return {"desc_offset": 0, "pitch": pitch, "labels_offset": labels_offset,
            "bytes": labels_offset + 4 * n_total}


def fused_gather_plan(n_total: int, rank: int, world: int, dim: int, multicast_ptr: int,
                      buffer_ptrs) -> dict:
    """lbp_extract_gather destinations of `rank`: MULTIMEM with the multicast address when it
    is non-zero, else PEERS with every rank's buffer address as mapped on this device."""
    from .lbpfused import LBP_GATHER_MAX_DST, LBP_GATHER_MULTIMEM, LBP_GATHER_PEERS
    lay = fused_gather_layout(n_total, dim)
    first, count = shard_range(n_total, rank, world)
    if multicast_ptr:
        mode, bases = LBP_GATHER_MULTIMEM, [int(multicast_ptr)]
    else:
        if len(buffer_ptrs) != world or world > LBP_GATHER_MAX_DST:
            raise ValueError("peer gather needs one mapped buffer per rank (world <= 8)")
        mode, bases = LBP_GATHER_PEERS, [int(p) for p in buffer_ptrs]
    return {"mode": mode, "bases": bases, "desc_offset": lay["desc_offset"],
            "pitch": lay["pitch"], "labels_offset": lay["labels_offset"], "row_base": first,
            "count": count, "bytes": lay["bytes"]}


class FusedDatabase:
    """The training matrix [n_total][dim] u16 + labels [n_total] int32 in symmetric memory
    (torch.distributed._symmetric_memory: one allocation per rank, mapped on every peer, plus
    the multicast mapping when NVLS is available).  `build()` extracts this rank's shard with
    lbp_extract_gather straight into every rank's copy, then runs the symmetric-memory barrier;
    after it every rank holds the whole database (global crop order)."""

    def __init__(self, n_total: int, dim: int, device, group=None):
        import torch.distributed._symmetric_memory as symm_mem
        self.group = group or dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.n_total, self.dim = n_total, dim
        lay = fused_gather_layout(n_total, dim)
        self.buf = symm_mem.empty(lay["bytes"], dtype=torch.uint8, device=device)
        self.handle = symm_mem.rendezvous(self.buf, self.group)
        ptrs = [int(p) for p in self.handle.buffer_ptrs]
        self.plan = fused_gather_plan(n_total, self.rank, self.world, dim,
                                      int(self.handle.multicast_ptr), ptrs)
        self.scratch = None

    @property
    def mode(self) -> str:
        from .lbpfused import LBP_GATHER_MULTIMEM
        return "multimem" if self.plan["mode"] == LBP_GATHER_MULTIMEM else "peers"

    def views(self):
        p = self.plan
        rows = self.buf[:self.n_total * p["pitch"] * 2].view(torch.uint16).view(
            self.n_total, p["pitch"])
        lab = self.buf[p["labels_offset"]:p["labels_offset"] + 4 * self.n_total].view(torch.int32)
        return rows[:, :self.dim], lab

    def build(self, grey, depth, rois, labels, dmin: int, dmax: int, cells_x: int, cells_y: int,
              bins: int, stream=None):
        from . import lbpfused
        p = self.plan
        if rois.shape[0] != p["count"]:
            raise ValueError(f"rank {self.rank}: {rois.shape[0]} ROIs, shard has {p['count']}")
        dst = lbpfused.gather_dst(p["mode"], p["bases"], p["desc_offset"], p["pitch"],
                                  p["labels_offset"] if labels is not None else -1, p["row_base"])
        if self.scratch is None or self.scratch.shape[0] < p["count"]:
            self.scratch = torch.empty((max(p["count"], 1), self.dim), dtype=torch.uint16,
                                       device=grey.device)
        s = stream if stream is not None else torch.cuda.current_stream(grey.device)
        lbpfused.lbp_extract_gather(grey, depth, rois, dmin, dmax, cells_x, cells_y, bins,
                                    labels, dst, scratch=self.scratch[:p["count"]], stream=s)
        with torch.cuda.stream(s):
            self.handle.barrier(channel=0)  # every rank's rows have landed everywhere
        return self.views()
