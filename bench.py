#!/usr/bin/env python
"""Benchmark of the fused-depth LBP descriptor + linear-SVM hot path (arXiv 1504.01883).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lbpfused|reference]

One step = the whole hot path (depth mask, LBP codes,
uniform bins, cell histograms, u16 descriptor, linear OvR SVM scores + labels)
over one batch of synthetic crops already resident in HBM.  The default
workload is BASELINE.json configs[2] ("config3"): 16,384 face crops of 128x128
grey u8 + depth u16 per GPU, 8x8 cells x 59 uniform bins, 100-identity SVM.
Multi-GPU (torchrun): every rank owns its own 16,384 crops (weak scaling, no
data-path collective); time = max over ranks.  Rank 0 prints one JSON line.

--impl reference times the CPU oracle (oracle/, plain single-threaded C, run on
T host threads over disjoint shards) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "face crops/sec (LBP+hist+SVM) at 1/2/4/8 B200; achieved HBM GB/s vs peak"
UNIT = "crops/s"

WORKLOADS = {
    # name: (crops per GPU, H, W, cells_x, cells_y, bins, classes, description)
    "config3": (16384, 128, 128, 8, 8, 59, 100,
                "BASELINE configs[2]: 16384 x 128x128 grey+depth crops with depth masks, "
                "8x8 cells x 59 uniform bins, 100-identity one-vs-all linear SVM"),
    "config4": (131072, 128, 128, 8, 8, 59, 1000,
                "BASELINE configs[3] shard: 131072 x 128x128 crops per GPU (2^20 over 8 GPUs), "
                "1000-identity SVM"),
    "config1": (1, 64, 64, 8, 8, 59, 2,
                "BASELINE configs[0]: single 64x64 grey+depth crop, 8x8x59, 2-class SVM"),
    "config2": (4, 128, 128, 8, 8, 59, 10,
                "BASELINE configs[1]: 640x480 Kinect-shaped grey+depth frame stream, 4 tracked "
                "faces (128x128 ROIs moving <= 20 px/frame), 10 identities"),
    # the tile variant of the TMA kernel (csrc/lbp_hist_tile.cuh): other crop sizes, batched
    "tile64": (16384, 64, 64, 8, 8, 59, 100,
               "16384 x 64x64 grey+depth crops (the crop size of BASELINE configs[0], batched), "
               "8x8 cells x 59 uniform bins, 100-identity one-vs-all linear SVM"),
    "tile100": (16384, 100, 100, 8, 8, 59, 100,
                "16384 x 100x100 grey+depth crops (SPEC's 100x100 ROI size; rows padded to 112 / "
                "208 B for TMA), 8x8 cells x 59 uniform bins, 100-identity SVM"),
    "tile200": (16384, 200, 200, 8, 8, 59, 100,
                "16384 x 200x200 grey+depth crops (the paper's resized face, P:154; grey rows "
                "padded to 208 B for TMA), 8x8 cells x 59 uniform bins, 100-identity SVM"),
    # crops = TOTAL database size (strong scaling: sharded over the ranks)
    "config5": (262144, 128, 128, 8, 8, 59, 0,
                "BASELINE configs[4]: online database build, 256k 128x128 crops sharded over the "
                "GPUs, descriptors + int32 labels all-gathered (NCCL) into the training matrix"),
    # training after the database build: crops = database size, 1 epoch
    "train": (16384, 128, 128, 8, 8, 59, 100,
              "SURVEY 8f-4: one-vs-rest linear SVM training (exact integer Pegasos) on a "
              "16384-crop database, 100 identities, 1 epoch"),
}
N_IDS = 100  # identities of the database build (label = crop index mod N_IDS)
DMIN, DMAX = 600, 1400


SOURCES = {"grey": 0, "depth": 1, "fused": 2}  # LBP_SRC_* of include/lbpfused.h


def bytes_per_crop(H, W, cx, cy, bins):
    """Algorithmic HBM bytes of the extraction kernel per crop:
    grey u8 + depth u16 read once, u16 descriptor written once."""
    return H * W * (1 + 2) + cx * cy * bins * 2


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="lbpfused", choices=["lbpfused", "reference"])
    p.add_argument("--workload", default="config3", choices=sorted(WORKLOADS))
    p.add_argument("--crops", type=int, default=0, help="override crops per GPU")
    p.add_argument("--dist", default="face", choices=["face", "constant", "noise"])
    p.add_argument("--no-depth", action="store_true")
    p.add_argument("--bins", type=int, default=0)
    p.add_argument("--source", default="grey", choices=sorted(SOURCES),
                   help="LBP code plane (configs 3/4): grey (headline), depth, or fused "
                        "grey||depth descriptor (SURVEY §8f-1)")
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--e2e-steps", type=int, default=0, help="0 = min(steps, 10)")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    p.add_argument("--skip-cpu", action="store_true")
    p.add_argument("--pipeline", action="store_true",
                   help="configs 3/4: score on a second stream so step k's scoring overlaps "
                        "step k+1's extraction (about 2.4%% more crops/s on config3; the "
                        "extraction launches then share the GPU, so their roofline fraction "
                        "reads lower -- off by default)")
    p.add_argument("--resize", type=int, default=0,
                   help="configs 1/2: resize every ROI to S x S on the GPU before the "
                        "descriptor (the paper's 200x200, P:154; lbp_extract_resized)")
    p.add_argument("--api", default="fused", choices=["fused", "split"],
                   help="configs 1/2: lbp_recognize (one fused cluster launch) or "
                        "lbp_fused_extract + svm_score (two launches)")
    p.add_argument("--chunks", type=int, default=4,
                   help="config5: extraction/all-gather overlap chunks (1 = serial)")
    p.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                   help="process-group backend for N > 1 (gloo: functional check only)")
    p.add_argument("--launch-check", action="store_true",
                   help="(tests) print each rank's RANK / WORLD_SIZE and exit")
    p.add_argument("--compact", action="store_true",
                   help="config5: all-gather u8 descriptors + exception lists (serial; "
                        "lbp_desc_pack_u8 / lbp_desc_unpack_u8), and time pack/unpack")
    p.add_argument("--format", default="auto", choices=["auto", "u8", "u16"],
                   help="descriptor between extraction and scoring (grey source): u8 = the "
                        "compact form (lbp_extract_u8 + svm_score_u8: u8 rows + records of the "
                        "entries above 255), u16 = lbp_fused_extract + svm_score; auto = the "
                        "faster step for the class count: u16 up to 124 classes (one TMEM "
                        "pass of the fp16 scorer: config3), u8 above (config4)")
    p.add_argument("--fused", action="store_true",
                   help="config5: the fused database build (SURVEY §8e way 2): the extraction "
                        "epilogue stores every row into every rank's symmetric-memory copy "
                        "(NVLS multicast when available, else NVLink peer stores) + one barrier")
    return p.parse_args()


# --------------------------------------------------------------------------- clocks (NVML)

class ClockSampler:
    """Polls SM clock and throttle reasons with NVML while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int, period_s: float = 0.0002):
        self.ok = False
        self.samples, self.reasons = [], set()
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            # the first query of each kind takes ~20 ms (tools/nvml_probe.py), the next ~1 us:
            # issue them here, outside the timed region
            pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML on this host
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            # the launching thread holds the GIL between its (GIL-releasing) ctypes calls;
            # with the default 5-ms switch interval the sampler would get a few samples per
            # timed region at most
            self._switch = sys.getswitchinterval()
            sys.setswitchinterval(1e-4)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()
            sys.setswitchinterval(self._switch)

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        busy = [s for s in self.samples]
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(busy)}


# --------------------------------------------------------------------------- CPU oracle

def oracle_rate(grey, depth, rois, W, b, cx, cy, bins, budget_s, threads, source=0):
    """Times the UNMODIFIED oracle (extraction + SVM) on T threads over disjoint shards of the
    sample, repeating passes over the sample until about `budget_s` seconds have elapsed.

    Returns (crops/s, crops processed, seconds, passes, descriptors, labels of one pass)."""
    import oracle
    n = grey.shape[0]
    shards = np.array_split(np.arange(n), threads)
    out_desc = [None] * threads
    out_lab = [None] * threads

    def work(i):
        idx = shards[i]
        if idx.size == 0:
            return
        dd = oracle.lbp_extract(grey[idx], depth[idx] if depth is not None else None,
                                _local_rois(rois[idx]), DMIN, DMAX, cx, cy, bins, source=source)
        _, lab, _ = oracle.svm_score(dd, W, b)
        out_desc[i], out_lab[i] = dd, lab

    passes, t0 = 0, time.perf_counter()
    while True:
        ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        passes += 1
        dt = time.perf_counter() - t0
        if dt >= budget_s or passes >= 1000:
            break
    desc = np.concatenate([x for x in out_desc if x is not None])
    lab = np.concatenate([x for x in out_lab if x is not None])
    return n * passes / dt, n * passes, dt, passes, desc, lab


def _local_rois(rois):
    r = np.array(rois, np.int32, copy=True)
    r[:, 0] = np.arange(r.shape[0])
    return r


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


# --------------------------------------------------------------------------- reference arm

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import synthgen
    n_gpu_crops, H, Wd, cx, cy, bins, C, desc_txt = WORKLOADS[args.workload]
    bins = args.bins or bins
    threads = len(os.sched_getaffinity(0))
    per_step = 256 * threads  # ~0.1 s of oracle work per step: thread start-up stays negligible
    total = per_step * (args.steps + args.warmup)
    grey, depth = synthgen.face_crops(per_step, H, Wd, seed=args.seed, dist=args.dist)
    if args.no_depth:
        depth = None
    rois = synthgen.full_rois(per_step, H, Wd)
    W, b = synthgen.svm_weights(C, cx * cy * bins, seed=args.seed)
    import oracle
    shards = np.array_split(np.arange(per_step), threads)

    def step():
        def work(idx):
            d = oracle.lbp_extract(grey[idx], None if depth is None else depth[idx],
                                   _local_rois(rois[idx]), DMIN, DMAX, cx, cy, bins)
            oracle.svm_score(d, W, b)
        ts = [threading.Thread(target=work, args=(s,)) for s in shards if s.size]
        for t in ts:
            t.start()
        for t in ts:
            t.join()

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    sample = (f"{per_step} crops per step ({desc_txt.split(':')[0]} crop shape), "
              f"{threads} threads x unmodified single-threaded oracle on disjoint shards")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(args, n_gpu_crops, H, Wd, cx, cy, bins, C, desc_txt),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, n, H, W, cx, cy, bins, C, desc_txt):
    return {"workload": f"{args.workload}: {desc_txt}", "crops_per_gpu": n, "crop": f"{H}x{W}",
            "cells": f"{cx}x{cy}", "bins": bins, "classes": C, "dist": args.dist,
            "depth_mask": not args.no_depth, "depth_window_mm": [DMIN, DMAX],
            "source": getattr(args, "source", "grey"),
            "descriptor": ("u8 + per-row records of counts > 255 (lbp_extract_u8 -> svm_score_u8)"
                           if compact_format(args) else "u16 (lbp_fused_extract -> svm_score)"),
            "parallelism": f"crop-sharded dp{int(os.environ.get('WORLD_SIZE', '1'))}",
            "pipeline": "scoring of step k overlaps extraction of step k+1 (2 streams)"
                        if getattr(args, "pipeline", False) else "serial",
            "l2": "inputs larger than L2 (no flush needed)" if n * H * W * 3 > 126e6 else
                  "inputs L2-resident (latency config)"}


def pad_rows(torch, t):
    """A view of t ([n][H][W]) in a buffer whose rows are a multiple of 16 B (TMA strides):
    200-px grey rows -> 208 B.  t itself when already aligned."""
    row = t.shape[-1] * t.element_size()
    if row % 16 == 0:
        return t
    P = (row + 15) // 16 * 16 // t.element_size()
    buf = torch.zeros((*t.shape[:-1], P), dtype=t.dtype, device=t.device,
                      pin_memory=(t.device.type == "cpu" and torch.cuda.is_available()))
    buf[..., :t.shape[-1]] = t
    return buf[..., :t.shape[-1]]


def compact_format(args) -> bool:
    """The recognition step runs on the compact descriptor (grey source only)."""
    return getattr(args, "format", "u16") == "u8" and getattr(args, "source", "grey") == "grey"


# --------------------------------------------------------------------------- own arm

def ensure_built():
    """Build the in-tree CUDA libraries if absent or stale (a no-op normally; concurrent ranks
    serialise on a lock file), before any timing."""
    from paper_1504_01883_b200 import build
    build.build()
    import synthgen
    synthgen.build_gpu()


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(args):
    """`bench.py --gpus N` (N > 1) run as a plain command: re-execute it under
    torch.distributed.run with N ranks (one process per GPU, rendezvous on 127.0.0.1), so the
    line reports the world size it measured.  Returns the launcher's exit code."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=dict(os.environ, LBP_BENCH_RELAUNCHED="1"))


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.launch_check:  # CPU test of the launcher: every rank reports what it sees
        # one write() per line: the ranks share the pipe and must not interleave
        sys.stdout.flush()
        os.write(1, (json.dumps({"rank": int(os.environ.get("RANK", "0")),
                                 "world": int(os.environ.get("WORLD_SIZE", "1")),
                                 "relaunched": os.environ.get("LBP_BENCH_RELAUNCHED") == "1"})
                     + "\n").encode())
        return 0
    if args.impl == "reference":
        return run_reference(args)
    ensure_built()
    if args.workload == "config5":
        return run_dbbuild(args)
    if args.workload == "train":
        return run_train(args)
    if args.workload in ("config1", "config2"):
        return run_latency(args)

    import torch
    import torch.distributed as dist

    import paper_1504_01883_b200 as lb
    import synthgen

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = rank_device(torch, local, world, args)
    if world > 1:
        init_dist(dist, args, dev)

    n, H, Wd, cx, cy, bins, C, desc_txt = WORKLOADS[args.workload]
    n = args.crops or n
    bins = args.bins or bins
    if args.format == "auto":
        args.format = "u16" if C <= 124 else "u8"
    source = SOURCES[args.source]
    if source != 0 and args.no_depth:
        raise SystemExit("--source depth/fused needs the depth plane")
    dim = cx * cy * bins * (2 if source == 2 else 1)
    first = rank * n  # global crop indices of this rank: [rank*n, (rank+1)*n)

    grey, depth = synthgen.gpu_face_crops(n, H, Wd, seed=args.seed, first_index=first,
                                          dist=args.dist, device=dev)
    grey = pad_rows(torch, grey)
    depth = pad_rows(torch, depth)
    if args.no_depth:
        depth = None
    rois = torch.from_numpy(synthgen.full_rois(n, H, Wd)).to(dev)
    W_np, b_np = synthgen.svm_weights(C, dim, seed=args.seed)
    W = torch.from_numpy(W_np).to(dev)
    b = torch.from_numpy(b_np).to(dev)
    compact = compact_format(args)
    prepared = lb.svm_prepare_u8(W) if compact else lb.svm_prepare(W)
    if compact:
        cap = lb.lbp_u8_exc_cap_min(lb.images_geometry(grey, depth), dim)
        desc = lb.CompactDesc.empty(n, dim, cap, dev)
    else:
        desc = torch.empty((n, dim), dtype=torch.uint16, device=dev)
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    top = torch.empty(n, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    # Step k = extraction of batch k then scoring of batch k.  With --pipeline the
    # scoring runs on a second stream, so step k's scoring overlaps step k+1's extraction
    # (descriptors double-buffered; the extraction of step k waits for the scoring of step
    # k-2, which read the same buffer).
    svm_stream = torch.cuda.Stream(dev) if args.pipeline else stream
    if args.pipeline:
        descs = [desc, lb.CompactDesc.empty(n, dim, desc.cap, dev) if compact
                 else torch.empty_like(desc)]
    else:
        descs = [desc, desc]
    ext_done = [torch.cuda.Event(), torch.cuda.Event()]
    svm_done = [torch.cuda.Event(), torch.cuda.Event()]
    step_no = [0]

    def step(ev=None):
        k = step_no[0]
        step_no[0] += 1
        buf = k & 1
        d_k = descs[buf]
        if args.pipeline and k >= 2:
            stream.wait_event(svm_done[buf])
        if ev is not None:
            ev[0].record(stream)
        if compact:
            lb.lbp_extract_u8(grey, depth, rois, DMIN, DMAX, cx, cy, bins, out=d_k,
                              stream=stream)
        elif source == 0:
            lb.lbp_fused_extract(grey, depth, rois, DMIN, DMAX, cx, cy, bins, out=d_k,
                                 stream=stream)
        else:
            lb.lbp_extract_source(grey, depth, rois, DMIN, DMAX, cx, cy, bins, source, out=d_k,
                                  stream=stream)
        if ev is not None:
            ev[1].record(stream)
        if args.pipeline:
            ext_done[buf].record(stream)
            svm_stream.wait_event(ext_done[buf])
        if ev is not None and not args.pipeline:
            ev[2].record(svm_stream)
        score = lb.svm_score_u8 if compact else lb.svm_score
        score(d_k, W, b, prepared=prepared, want_scores=False, labels=labels, top_score=top,
              stream=svm_stream)
        if ev is not None and not args.pipeline:
            ev[3].record(svm_stream)
        if args.pipeline:
            svm_done[buf].record(svm_stream)

    launches_per_step = 3 if source == 2 else 2  # extraction kernel(s) + svm_gemm
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, barrier + sync on both sides, events on the launching stream.
    # The headline pass records no event between the kernels (an event between the extraction
    # and the scorer would cut the programmatic dependent launch that overlaps the scorer's
    # prologue with the extraction's tail); a second pass of K steps with events around each
    # kernel gives the per-kernel durations of the roofline lines.
    ev_ext = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(4))
              for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # clocks are sampled through both timed passes (the headline K steps, then the same K
    # steps with events around each kernel): a 20-step config3 region alone is ~5 ms
    with ClockSampler(torch.cuda.current_device()) as clk:
        t_start.record(stream)
        for k in range(args.steps):
            step()
        stream.wait_stream(svm_stream)  # the last step's scoring is inside the timed region
        t_end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = t_start.elapsed_time(t_end)
        # per-kernel pass (same K steps, events around each launch)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            step(ev_ext[k])
        stream.wait_stream(svm_stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ext_ms = sum(e[0].elapsed_time(e[1]) for e in ev_ext) / args.steps
    svm_ms = (sum(e[2].elapsed_time(e[3]) for e in ev_ext) / args.steps
              if not args.pipeline else float("nan"))
    t = torch.tensor([ms, ext_ms, svm_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, ext_ms, svm_ms = float(t[0]), float(t[1]), float(t[2])
    ms_per_step = ms / args.steps
    value = n * world / (ms_per_step * 1e-3)

    # ---- end to end through the public C ABI from pinned HOST buffers
    e2e = None
    if source == 0:  # lbp_recognize_host computes the grey-source descriptor
        e2e = run_e2e(args, lb, torch, dist, world, dev, grey, depth, H, Wd, cx, cy, bins, W, b,
                      lb.svm_prepare(W) if compact else prepared, n)

    # ---- roofline of the dominant kernel (lbp_hist): algorithmic bytes / avg launch time
    peaks = load_peaks()
    if compact:  # grey + depth read, u8 row + its exception count written (records: ~0)
        bpc = (H * Wd * 3 if depth is not None else H * Wd) + dim + 4
    elif source == 0:
        bpc = bytes_per_crop(H, Wd, cx, cy, bins) if depth is not None else H * Wd + dim * 2
    elif source == 1:
        bpc = H * Wd * 2 + dim * 2  # depth read once (mask + codes), descriptor written
    else:
        bpc = H * Wd * 3 + dim * 2  # grey + depth read once, both blocks written
    achieved = bpc * n / (ext_ms * 1e-3) / 1e9
    peak, peak_src = peaks
    roofline = {"bound": "hbm", "kernel": "lbp_hist (extraction)" if source == 0 else
                "extraction (" + args.source + " source)", "achieved": achieved,
                "peak": peak, "unit": "GB/s", "frac": achieved / peak if peak else None,
                "peak_source": peak_src, "bytes_per_crop": bpc,
                "frac_of_nominal_8000": achieved / 8000.0,  # also vs 8 TB/s
                "kernel_ms": ext_ms, "kernel_share_of_step": ext_ms / ms_per_step,
                "traffic": load_traffic(args.workload, bins, args.source,
                                        depth is not None and not args.no_depth,
                                        "u8" if compact else "u16")}
    # the scorer's own roofline (per-phase TF/s fractions): algorithmic flops
    # 2 n C dim of s = W x + b over its event-timed launch; the INT8 digit-plane kernel
    # (C > 124) takes the int8 peak = the measured bf16 burst x the nominal 2x ratio
    if not args.pipeline and prepared is not None:
        flops = 2.0 * n * C * dim
        i8 = C > 124 or compact
        bf16 = load_bf16_peak()
        pk = bf16 * (2.0 if i8 else 1.0)
        ach = flops / (svm_ms * 1e-3) / 1e12
        roofline["scorer"] = {
            "bound": "tensor", "kernel": "svm_gemm_u8 (INT8 digit planes, u8 descriptors by "
            "TMA)" if compact else "svm_gemm_i8 (INT8 digit planes)" if i8 else
            "svm_gemm (fp16 digit planes)", "achieved": ach, "unit": "TFLOP/s",
            "peak": pk, "frac": ach / pk, "frac_of_bf16_burst": ach / bf16,
            "peak_source": ("MEASURED_PEAKS.json bf16_tflops x 2 (nominal int8:bf16 ratio)"
                            if i8 else "MEASURED_PEAKS.json bf16_tflops (burst)"),
            "flops_per_step": flops, "kernel_ms": svm_ms,
            "kernel_share_of_step": svm_ms / ms_per_step}

    # ---- CPU oracle baseline (rank 0, N=1 only) + equivalence gate on its sample
    cpu = None
    gate_m = 4096 if world == 1 else 512
    last = descs[(step_no[0] - 1) & 1]
    gscores, gtop, same = gate_scores(lb, torch, last, W, b, prepared, labels, top,
                                      min(gate_m, n))
    if not same:
        print(json.dumps({"error": "scorer with scores requested disagrees with the timed step"}),
              flush=True)
        return 3
    if rank == 0 and world == 1 and not args.skip_cpu:
        cpu, gate_ok = run_cpu_leg(args, torch, grey, depth, rois, last, labels, W_np, b_np,
                                   cx, cy, bins, gscores, gtop)
        if not gate_ok:
            print(json.dumps({"error": "equivalence gate failed: GPU != oracle on the sample"}),
                  flush=True)
            return 3
    elif world > 1:  # every rank checks its own shard's first crops; any failure stops all
        ok = rank_gate(torch, grey, depth, rois, last, labels, W_np, b_np, cx, cy, bins, source,
                       512, gscores, gtop)
        flag = torch.tensor([1 if ok else 0], device=dev, dtype=torch.int32)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag[0]) == 0:
            if rank == 0:
                print(json.dumps({"error": "equivalence gate failed on some rank"}), flush=True)
            return 3

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": workload_config(args, n, H, Wd, cx, cy, bins, C, desc_txt),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(),
            "timing": "ms_per_step: K steps between two events (no event between kernels); "
                      "kernel_ms: a second pass of the same K steps with events around each "
                      "kernel",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_latency(args):
    """Configs 1 and 2 are latency cases (one 64x64 crop; one 640x480 frame with 4 faces):
    per-call device latency of extraction + SVM, eager (p50/p99 over calls, CUDA events) and
    as a replayed CUDA graph of all calls (throughput).  Inputs are device-resident."""
    import torch

    import paper_1504_01883_b200 as lb
    import synthgen
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n_per, H, Wd, cx, cy, bins, C, desc_txt = WORKLOADS[args.workload]
    if args.workload == "config1":
        n_calls = 256
        g, d = synthgen.face_crops(n_calls, 64, 64, seed=args.seed)
        rois_np = synthgen.full_rois(n_calls, 64, 64)
        frame_bytes = 64 * 64 * 3
    else:
        n_calls = 240
        g, d, rois_np = synthgen.kinect_frames(n_calls, seed=args.seed)
        frame_bytes = 640 * 480 * 3
    grey = torch.from_numpy(g).to(dev)
    depth = torch.from_numpy(d.view(np.int16)).to(dev).view(torch.uint16)
    rois = torch.from_numpy(rois_np).to(dev)
    dim = cx * cy * bins
    W_np, b_np = synthgen.svm_weights(C, dim, seed=args.seed)
    W, b = torch.from_numpy(W_np).to(dev), torch.from_numpy(b_np).to(dev)
    prepared = lb.svm_prepare(W)
    desc = torch.empty((n_calls * n_per, dim), dtype=torch.uint16, device=dev)
    labels = torch.empty(n_calls * n_per, dtype=torch.int32, device=dev)
    top = torch.empty(n_calls * n_per, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)

    fused = args.api == "fused" and not args.resize

    def call(f):
        r = rois[f * n_per:(f + 1) * n_per]
        o = desc[f * n_per:(f + 1) * n_per]
        if fused:  # one launch: cluster of cells_y CTAs per ROI, extraction + SVM via DSMEM
            lb.lbp_recognize(grey, depth, r, DMIN, DMAX, cx, cy, bins, W, b, prepared=prepared,
                             desc=o, labels=labels[f * n_per:(f + 1) * n_per],
                             top_score=top[f * n_per:(f + 1) * n_per], stream=stream)
            return
        if args.resize:
            lb.lbp_extract_resized(grey, depth, r, args.resize, DMIN, DMAX, cx, cy, bins,
                                   out=o, stream=stream)
        else:
            lb.lbp_fused_extract(grey, depth, r, DMIN, DMAX, cx, cy, bins, out=o, stream=stream)
        lb.svm_score(o, W, b, prepared=prepared, want_scores=False,
                     labels=labels[f * n_per:(f + 1) * n_per],
                     top_score=top[f * n_per:(f + 1) * n_per], stream=stream)

    with torch.cuda.stream(stream):
        for f in range(min(8, n_calls)):
            call(f)
    torch.cuda.synchronize()
    # eager: one call at a time, events on the launching stream
    lat = []
    for f in range(n_calls):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        call(f)
        z.record(stream)
        z.synchronize()
        lat.append(a.elapsed_time(z))
    lat = np.array(lat)
    # graph: all calls captured once, replayed
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        for f in range(n_calls):
            call(f)
    graph.replay()
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(args.steps // 10, 3)
    with ClockSampler(0) as clk, torch.cuda.stream(stream):  # replay() launches on the
        a.record(stream)                                     # current stream
        for _ in range(reps):
            graph.replay()
        z.record(stream)
        torch.cuda.synchronize()
    per_call_graph = a.elapsed_time(z) / reps / n_calls
    # batched: every call's ROIs in one extraction + one scoring launch (a frame buffer
    # processed as a batch; >= 148 ROIs take the persistent TMA kernel)
    def batched():
        lb.lbp_fused_extract(grey, depth, rois, DMIN, DMAX, cx, cy, bins, out=desc, stream=stream)
        lb.svm_score(desc, W, b, prepared=prepared, want_scores=False, labels=labels,
                     top_score=top, stream=stream)
    with torch.cuda.stream(stream):
        for _ in range(3):
            batched()
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            batched()
        z.record(stream)
        torch.cuda.synchronize()
    per_batch = a.elapsed_time(z) / reps
    line = {
        "metric": METRIC, "value": n_per / (per_call_graph * 1e-3), "unit": UNIT, "n_gpus": 1,
        "steps": reps * n_calls, "warmup": 8, "ms_per_step": per_call_graph,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": f"{args.workload}: {desc_txt}", "crops_per_call": n_per,
                   "calls": n_calls, "classes": C, "l2": "inputs L2-resident (latency config)",
                   "resize": args.resize or None},
        "latency_us": {"eager_p50": float(np.percentile(lat, 50) * 1e3),
                       "eager_p99": float(np.percentile(lat, 99) * 1e3),
                       "graph_per_call": per_call_graph * 1e3},
        "batched": {"calls": n_calls, "crops": n_calls * n_per, "us_per_batch": per_batch * 1e3,
                    "crops_per_s": n_calls * n_per / (per_batch * 1e-3)},
        "frame_h2d_bytes": frame_bytes, "gpu_launches": (1 if fused else 2) * n_calls * reps,
        "api": "lbp_recognize (fused)" if fused else "lbp_fused_extract/lbp_extract_resized + "
               "svm_score", "clocks": clk.summary(),
        "roofline": None, "cpu_baseline": latency_cpu_leg(args, g, d, rois_np, n_per, W_np, b_np,
                                                          cx, cy, bins), "e2e": None,
    }
    print(json.dumps(line), flush=True)
    return 0


def latency_cpu_leg(args, g, d, rois_np, n_per, W_np, b_np, cx, cy, bins):
    """The oracle, single-threaded, on the first calls of the latency workload (ms per call)."""
    if args.skip_cpu:
        return None
    import oracle
    calls = 16
    t0 = time.perf_counter()
    for f in range(calls):
        r = rois_np[f * n_per:(f + 1) * n_per]
        if args.resize:
            dd = oracle.lbp_extract_resized(g, d, r, args.resize, DMIN, DMAX, cx, cy, bins)
        else:
            dd = oracle.lbp_extract(g, d, r, DMIN, DMAX, cx, cy, bins)
        oracle.svm_score(dd, W_np, b_np)
    ms = (time.perf_counter() - t0) / calls * 1e3
    return {"value": n_per / (ms * 1e-3), "unit": UNIT, "cores": 1, "kind": "oracle",
            "ms_per_call": ms, "sample": f"first {calls} calls, one thread", "cpu": cpu_model()}


def run_dbbuild(args):
    """Config 5: each rank extracts its shard of the database, then an all-gather over NCCL
    assembles the full [N][dim] u16 training matrix and labels on every rank.  One step =
    extraction + all-gather of all N crops; value = N / step time (strong scaling)."""
    import torch
    import torch.distributed as dist

    import paper_1504_01883_b200 as lb
    import synthgen
    from paper_1504_01883_b200.parallel import (gather_database, gather_database_chunked,
                                                gather_database_compact,
                                                shard_range)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = rank_device(torch, local, world, args)
    if world > 1:
        init_dist(dist, args, dev)
    else:  # the gather is a no-op copy; keep one code path with a 1-rank gloo group
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + (os.getpid() % 1000)))
        dist.init_process_group("gloo" if not torch.cuda.is_available() else "nccl",
                                rank=0, world_size=1, device_id=dev)
    n_total, H, Wd, cx, cy, bins, _, desc_txt = WORKLOADS["config5"]
    n_total = args.crops or n_total
    first, count = shard_range(n_total, rank, world)
    grey, depth = synthgen.gpu_face_crops(count, H, Wd, seed=args.seed, first_index=first,
                                          dist=args.dist, device=dev)
    rois = torch.from_numpy(synthgen.full_rois(count, H, Wd)).to(dev)
    labels = (torch.arange(first, first + count, device=dev) % N_IDS).to(torch.int32)
    dim = cx * cy * bins
    desc = torch.empty((count, dim), dtype=torch.uint16, device=dev)
    stream = torch.cuda.current_stream(dev)

    comm = torch.cuda.Stream(dev)
    if args.compact or args.fused:
        args.chunks = 1  # serial exchanges: extract (+ pack), exchange (+ unpack)
    fdb = None
    if args.fused:
        from paper_1504_01883_b200.parallel import FusedDatabase
        fdb = FusedDatabase(n_total, dim, dev)

    def extract_chunk(lo, hi):
        lb.lbp_fused_extract(grey, depth, rois[lo:hi], DMIN, DMAX, cx, cy, bins,
                             out=desc[lo:hi], stream=stream)
        return desc[lo:hi]

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        if fdb is not None:  # one kernel writes every rank's copy, then the barrier
            full, lab = fdb.build(grey, depth, rois, labels, DMIN, DMAX, cx, cy, bins,
                                  stream=stream)
            if ev is not None:
                ev[1].record(stream)
                ev[2].record(stream)
            return full, lab
        if args.chunks <= 1:  # serial: extract everything, then one all-gather
            lb.lbp_fused_extract(grey, depth, rois, DMIN, DMAX, cx, cy, bins, out=desc,
                                 stream=stream)
            if ev is not None:
                ev[1].record(stream)
            if args.compact:
                full, lab = gather_database_compact(desc, labels, n_total)
            else:
                full, lab = gather_database(desc, labels, n_total)
        else:  # chunked: chunk k's all-gather overlaps chunk k+1's extraction
            if ev is not None:
                ev[1].record(stream)
            full, lab = gather_database_chunked(extract_chunk, labels, n_total, dim, args.chunks,
                                                device=dev, comm_stream=comm)
        if ev is not None:
            ev[2].record(stream)
        return full, lab

    for _ in range(max(args.warmup, 3)):
        full, lab = step()
    torch.cuda.synchronize()
    evs = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0 = time.perf_counter()
        for k in range(args.steps):
            full, lab = step(evs[k])
        torch.cuda.synchronize()
    dist.barrier()
    ext = sum(a.elapsed_time(b) for a, b, _ in evs) / args.steps
    gat = sum(b.elapsed_time(c) for _, b, c in evs) / args.steps
    tot = evs[0][0].elapsed_time(evs[-1][2]) / args.steps
    t = torch.tensor([tot, ext, gat], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot, ext, gat = (float(v) for v in t)
    gathered = n_total * dim * (1 if args.compact else 2) + n_total * 4
    compact = None
    if args.compact:  # the pack / unpack kernels alone on this rank's shard (HBM-bound)
        packed, exc, cnt = lb.desc_pack_u8(desc, row_base=first, cap=4096)
        out16 = torch.empty_like(desc)
        reps = 10
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        e[0].record(stream)
        for _ in range(reps):
            lb.desc_pack_u8(desc, row_base=first, cap=4096, packed=packed, exc=exc, count=cnt)
        e[1].record(stream)
        for _ in range(reps):
            lb.desc_unpack_u8(packed, exc, cnt, 4096, row_base=first, out=out16)
        e[2].record(stream)
        torch.cuda.synchronize()
        pk, up = e[0].elapsed_time(e[1]) / reps, e[1].elapsed_time(e[2]) / reps
        entries = count * dim
        compact = {"pack_ms": pk, "unpack_ms": up, "exceptions": int(cnt.item()),
                   "pack_GBps": 3 * entries / (pk * 1e-3) / 1e9,
                   "unpack_GBps": 3 * entries / (up * 1e-3) / 1e9,
                   "roundtrip_exact": bool(torch.equal(out16.view(torch.int16),
                                                       desc.view(torch.int16))),
                   "note": "bytes per entry: pack 2 read + 1 written, unpack 1 + 2; the "
                           "all-gather moves 1 B per entry + 16 B per exception"}
    if args.chunks > 1:  # phases overlap: no separate phase times; bound both by the step
        ext = gat = tot
    peak, peak_src = load_peaks()
    bpc = bytes_per_crop(H, Wd, cx, cy, bins)
    if rank == 0:
        line = {
            "metric": METRIC, "value": n_total / (tot * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": tot,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": {"workload": f"config5: {desc_txt}", "crops_total": n_total,
                       "crops_per_gpu": count, "crop": f"{H}x{Wd}", "cells": f"{cx}x{cy}",
                       "bins": bins, "n_ids": N_IDS, "parallelism": f"crop-sharded dp{world} + "
                       + (f"fused gather ({fdb.mode} stores from the extraction epilogue)"
                          if fdb is not None else "all-gather")},
            "extract_ms": ext if args.chunks <= 1 else None,
            "allgather_ms": gat if args.chunks <= 1 else None,
            "overlap": {"chunks": args.chunks, "note": "chunk k's all-gather on a second stream "
                        "overlaps chunk k+1's extraction" if args.chunks > 1 else "serial"},
            "compact": compact,
            "allgather": {"bytes_out_per_rank": gathered,
                          # one rank moves nothing: no bandwidth to report
                          "algbw_GBps": gathered / (gat * 1e-3) / 1e9
                          if gat > 0 and world > 1 and args.chunks <= 1 else None,
                          "busbw_GBps": gathered * (world - 1) / world / (gat * 1e-3) / 1e9
                          if gat > 0 and world > 1 and args.chunks <= 1 else None},
            "roofline": {"bound": "hbm", "kernel": "lbp_hist (extraction)",
                         "achieved": bpc * count / (ext * 1e-3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": bpc * count / (ext * 1e-3) / 1e9 / peak,
                         "peak_source": peak_src, "traffic": None},
            "cpu_baseline": None, "e2e": None,
            "gpu_launches": args.steps * (2 if fdb is not None else max(1, args.chunks) +
                                            (3 if args.compact and world > 1 else 0)),
            "clocks": clk.summary(),
            "check": {"rows": int(full.shape[0]), "label_ok": bool(
                (lab.cpu() == (torch.arange(n_total) % N_IDS).to(torch.int32)).all()),
                "desc_sample_ok": db_sample_ok(full, n_total, H, Wd, cx, cy, bins, args)},
        }
        if not (line["check"]["label_ok"] and line["check"]["desc_sample_ok"]):
            print(json.dumps({"error": "database check failed", "check": line["check"]}),
                  flush=True)
            dist.destroy_process_group()
            return 3
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def run_train(args):
    """SVM training on the GPU: descriptors of a synthetic database, then
    svm_train_ovr over one seeded epoch; rate = training steps (sample x class) per second.
    The oracle trains the same classes on the same inputs for a bounded sample of classes
    (equivalence gate: the integer state must match bit for bit)."""
    import torch

    import paper_1504_01883_b200 as lb
    import synthgen
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n, H, Wd, cx, cy, bins, C, desc_txt = WORKLOADS["train"]
    n = args.crops or n
    grey, depth = synthgen.gpu_face_crops(n, H, Wd, seed=args.seed, device=dev)
    rois = torch.from_numpy(synthgen.full_rois(n, H, Wd)).to(dev)
    desc = lb.lbp_fused_extract(grey, depth, rois, DMIN, DMAX, cx, cy, bins)
    labels = (torch.arange(n, device=dev) % C).to(torch.int32)
    order = torch.from_numpy(synthgen.train_order(n, 1, seed=args.seed)).to(dev)
    inv_lambda = 10000
    lb.svm_train_ovr(desc, labels, C, order[:min(n, 256)], inv_lambda)  # warm-up
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        a.record(stream)
        W, b, zst = lb.svm_train_ovr(desc, labels, C, order, inv_lambda, return_z=True)
        z.record(stream)
        torch.cuda.synchronize()
    ms = a.elapsed_time(z)
    steps = n * C
    cpu = None
    if not args.skip_cpu:
        import oracle
        k = 2  # classes timed on the host (one thread), same inputs
        dn = desc.cpu().view(torch.int16).numpy().view(np.uint16)
        t0 = time.perf_counter()
        _, _, zr = oracle.svm_train_ovr(dn, labels.cpu().numpy(), k, order.cpu().numpy(),
                                        inv_lambda, return_z=True)
        secs = time.perf_counter() - t0
        gate = bool(np.array_equal(zst[:k].cpu().numpy(), zr))
        cpu = {"value": n * k / secs, "unit": "training steps/s", "cores": 1, "kind": "oracle",
               "sample": f"{k} of {C} classes, one epoch of {n} samples, one thread, {secs:.1f} s",
               "equivalence_gate": "pass" if gate else "FAIL"}
        if not gate:
            print(json.dumps({"error": "equivalence gate failed: GPU training != oracle"}))
            return 3
    line = {"metric": "SVM training steps (sample x class) per second", "value": steps / (ms * 1e-3),
            "unit": "training steps/s", "n_gpus": 1, "steps": 1, "warmup": 1, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic",
            "config": {"workload": f"train: {desc_txt}", "samples": n, "classes": C,
                       "epochs": 1, "dim": cx * cy * bins, "inv_lambda": inv_lambda},
            "cpu_baseline": cpu, "e2e": None, "gpu_launches": 1, "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    return 0


def run_e2e(args, lb, torch, dist, world, dev, grey, depth, H, Wd, cx, cy, bins, W, b, prepared, n):
    """Same metric through lbp_recognize_host: H2D of the step's inputs from pinned host memory,
    extraction + SVM, D2H of labels and top scores, every step."""
    import synthgen
    steps = args.e2e_steps or min(args.steps, 10)
    g_h = pad_rows(torch, grey.cpu()) if grey.stride(1) != grey.shape[2] else grey.cpu().pin_memory()
    if not g_h.is_pinned():
        g_h = g_h.pin_memory()
    d_h = None
    if depth is not None:
        d_h = pad_rows(torch, depth.cpu()) if depth.stride(1) != depth.shape[2] else depth.cpu()
        if not d_h.is_pinned():
            d_h = d_h.pin_memory()
    r_h = torch.from_numpy(synthgen.full_rois(n, H, Wd)).pin_memory()
    lab_h = torch.empty(n, dtype=torch.int32).pin_memory()
    top_h = torch.empty(n, dtype=torch.float32).pin_memory()
    geom = lb.images_geometry(g_h, d_h)
    ws = torch.empty(lb.lbp_recognize_workspace_bytes(geom, d_h is not None, n, cx, cy, bins),
                     dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        lb.lbp_recognize_host(g_h, d_h, r_h, DMIN, DMAX, cx, cy, bins, W, b, prepared, ws, lab_h,
                              top_h, stream=stream)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        step()
    z.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(z) / steps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    # bytes the call copies: whole images including any row padding
    h2d = (g_h.untyped_storage().nbytes() +
           (d_h.untyped_storage().nbytes() if d_h is not None else 0) + r_h.numel() * 4)
    return {"value": n * world / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "steps": steps,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(n * 8),
            "api": "lbp_recognize_host (C ABI, pinned host buffers)"}


def run_cpu_leg(args, torch, grey, depth, rois, desc, labels, W_np, b_np, cx, cy, bins,
                gscores=None, gtop=None):
    """Oracle timed on this host's cores on a bounded sample; the sample's oracle output is
    also the equivalence gate (descriptors bit-exact, scores within R13, labels equal away
    from ties)."""
    threads = len(os.sched_getaffinity(0))
    n = grey.shape[0]
    m = min(n, 4096)
    g = np.ascontiguousarray(grey[:m].cpu().numpy())
    d = depth[:m].cpu().view(torch.int16).numpy().view(np.uint16) if depth is not None else None
    r = rois[:m].cpu().numpy()
    rate, done, secs, passes, odesc, olab = oracle_rate(g, d, r, W_np, b_np, cx, cy, bins,
                                                        args.cpu_seconds, threads,
                                                        SOURCES[args.source])
    gdesc = desc_rows(torch, desc, m)
    glab = labels[:m].cpu().numpy()
    ok, detail = gate_compare(gdesc, glab, odesc, olab, W_np, b_np,
                              None if gscores is None else gscores[:m],
                              None if gtop is None else gtop[:m])
    # SURVEY §8(d) also asks for the single-threaded oracle: one thread, first 256 crops
    r1, _, s1, _, _, _ = oracle_rate(g[:256], d[:256] if d is not None else None, r[:256], W_np,
                                     b_np, cx, cy, bins, 2.0, 1, SOURCES[args.source])
    cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
           "sample": f"first {m} crops of this workload x {passes} passes = {done} crops "
                     f"(extraction + SVM), {threads} threads x unmodified single-threaded C "
                     f"oracle on disjoint shards, {secs:.1f} s",
           "single_thread_value": r1,
           "cpu": cpu_model(), "equivalence_gate": "pass" if ok else "FAIL",
           "gate_detail": detail}
    return cpu, ok


def db_sample_ok(full, n_total, H, Wd, cx, cy, bins, args, k=8):
    """The gathered database against the oracle on k rows spread over every rank's shard
    (crop i is a pure function of its global index, so rank 0 regenerates it)."""
    import oracle
    import synthgen
    import torch
    idx = np.unique(np.linspace(0, n_total - 1, k).astype(np.int64))
    for i in idx:
        g, d = synthgen.face_crops(1, H, Wd, seed=args.seed, first_index=int(i), dist=args.dist)
        ref = oracle.lbp_extract(g, d, synthgen.full_rois(1, H, Wd), DMIN, DMAX, cx, cy, bins)
        got = full[int(i)].cpu().view(torch.int16).numpy().view(np.uint16)
        if not np.array_equal(got, ref[0]):
            return False
    return True


def gate_compare(gdesc, glab, odesc, olab, W_np, b_np, gscores=None, gtop=None):
    """Equivalence gate: descriptors bit-exact; scores and top scores within R13 and labels equal
    away from ties (R14) -- the one definition in oracle/tolerance.py, shared with the tests and
    smoke()."""
    if not np.array_equal(gdesc, odesc):
        return False, {"descriptors": "mismatch"}
    import oracle
    from oracle.tolerance import check_svm
    s_ref, _, _ = oracle.svm_score(odesc, W_np, b_np)
    ok, detail = check_svm(odesc, W_np, b_np, s_ref, olab, glab, s_gpu=gscores, top_gpu=gtop)
    detail["descriptors"] = "bit-exact"
    return ok, detail


def desc_rows(torch, desc, m):
    """The first m descriptor rows as numpy u16: a u16 tensor, or a CompactDesc decoded on the
    host (u8 entries, then each row's records of the counts above 255)."""
    if isinstance(desc, torch.Tensor):
        return desc[:m].cpu().view(torch.int16).numpy().view(np.uint16)
    out = desc.packed[:m].cpu().numpy().astype(np.uint16)
    n_exc = desc.exc_n[:m].cpu().numpy()
    exc = desc.exc[:m].cpu().numpy().view(np.uint32)
    for i in np.nonzero(n_exc)[0]:
        for k in range(min(int(n_exc[i]), exc.shape[1])):
            out[i, exc[i, k] >> 16] = exc[i, k] & 0xFFFF
    return out


def gate_scores(lb, torch, desc, W, b, prepared, labels, top, m):
    """Scores of the gate sample from the scorer in the bench's launch configuration (the whole
    batch, scores requested).  u16 path: its labels / top scores must equal the timed step's
    bit for bit.  Compact path: the timed step ran the label-only scorer (4 digit planes, a
    per-row proof, exact fix-up), so the gate checks the timed step's own labels and top
    scores against the oracle (returned here) and the scores-mode scores separately."""
    compact = not isinstance(desc, torch.Tensor)
    score = lb.svm_score_u8 if compact else lb.svm_score
    s_full, lab_full, top_full = score(desc, W, b, prepared=prepared, want_scores=True)
    torch.cuda.synchronize()
    if compact:
        return s_full[:m].cpu().numpy(), top[:m].cpu().numpy(), bool((labels >= -1).all())
    same = bool(torch.equal(lab_full, labels)) and bool(
        torch.equal(top_full.view(torch.int32), top.view(torch.int32)))
    return s_full[:m].cpu().numpy(), top_full[:m].cpu().numpy(), same


def rank_gate(torch, grey, depth, rois, desc, labels, W_np, b_np, cx, cy, bins, source, m,
              gscores=None, gtop=None):
    """The equivalence gate on every rank at N > 1 (no CPU timing): the oracle on this
    rank's first m crops."""
    import oracle
    m = min(m, grey.shape[0])
    g = np.ascontiguousarray(grey[:m].cpu().numpy())
    d = depth[:m].cpu().view(torch.int16).numpy().view(np.uint16) if depth is not None else None
    r = rois[:m].cpu().numpy()
    odesc = oracle.lbp_extract(g, d, r, DMIN, DMAX, cx, cy, bins, source=source)
    _, olab, _ = oracle.svm_score(odesc, W_np, b_np)
    gdesc = desc_rows(torch, desc, m)
    ok, _ = gate_compare(gdesc, labels[:m].cpu().numpy(), odesc, olab, W_np, b_np,
                         None if gscores is None else gscores[:m],
                         None if gtop is None else gtop[:m])
    return ok


def rank_device(torch, local, world, args):
    """cuda:LOCAL_RANK (one process per GPU).  --dist-backend gloo lets several ranks share
    a device (a functional check of the multi-rank code path on a one-GPU box: nothing in the
    timed path waits on another rank's kernels; such a run is never a measurement)."""
    idx = local if args.dist_backend == "nccl" else local % torch.cuda.device_count()
    torch.cuda.set_device(idx)
    return torch.device("cuda", idx)


def init_dist(dist, args, dev):
    if args.dist_backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def load_bf16_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
    except Exception:
        return 1590.0  # B200_PROFILING.md fallback


def load_traffic(workload, bins=59, source="grey", depth=True, fmt="u16"):
    """dram read+write bytes per launch of the extraction kernel from the committed ncu
    --set full capture of exactly this workload, bin count, code source, mask and descriptor
    format (None when no capture of that combination is committed)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    key = f"{workload}/bins{bins}/{source}/{'mask' if depth else 'nomask'}/{fmt}"
    try:
        return json.load(open(p)).get(key)
    except Exception:
        return None


if __name__ == "__main__":
    sys.exit(main())
