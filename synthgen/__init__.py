"""Seeded synthetic Kinect-shaped inputs (grey u8 + depth u16 face crops, SVM weights).

This module is the ONLY code shared by the oracle side (tests / bench cpu leg)
and the CUDA side.  It holds none of the method's arithmetic (no LBP codes, no
histograms, no SVM scores): it only draws inputs.  The recipe is DESIGN.md §4.

Every sample is a pure function of (seed, global crop index, y, x) through a
counter-based integer hash, so crop i is bit-identical whichever rank or batch
produces it.  ``synthgen/synth_gen.cu`` implements the same integer recipe on
the GPU for large batches; tests/test_synth_gpu.py checks the two bit-exactly.
"""
from __future__ import annotations

import numpy as np

DIST_FACE, DIST_CONSTANT, DIST_NOISE = 0, 1, 2
DISTS = {"face": DIST_FACE, "constant": DIST_CONSTANT, "noise": DIST_NOISE}

# default depth window (mm) of the synthetic workload: face at ~1 m
DMIN, DMAX = 600, 1400

_M1 = np.uint32(0x7FEB352D)
_M2 = np.uint32(0x846CA68B)
_GOLD = np.uint32(0x9E3779B9)


def _lowbias32(x):
    x = x.astype(np.uint32, copy=True)
    x ^= x >> np.uint32(16)
    x *= _M1
    x ^= x >> np.uint32(15)
    x *= _M2
    x ^= x >> np.uint32(16)
    return x


def hash5(seed, n, a, b, salt):
    """32-bit counter hash of (seed, crop index n, a, b, salt); numpy broadcasting."""
    with np.errstate(over="ignore"):
        h = _lowbias32(np.asarray(np.uint32(seed) + _GOLD * np.uint32(salt), dtype=np.uint32))
        h = _lowbias32(h ^ np.asarray(n, dtype=np.uint64).astype(np.uint32))
        h = _lowbias32(h ^ np.asarray(a, dtype=np.int64).astype(np.uint32))
        h = _lowbias32(h ^ np.asarray(b, dtype=np.int64).astype(np.uint32))
    return h


def _value_noise(seed, n, y, x, shift, mask, salt):
    """Integer bilinear value noise on a 2^shift lattice; returns int64 in [0, mask]."""
    cell = 1 << shift
    Y, X = y >> shift, x >> shift
    fy, fx = y & (cell - 1), x & (cell - 1)
    v00 = (hash5(seed, n, Y, X, salt) & mask).astype(np.int64)
    v01 = (hash5(seed, n, Y, X + 1, salt) & mask).astype(np.int64)
    v10 = (hash5(seed, n, Y + 1, X, salt) & mask).astype(np.int64)
    v11 = (hash5(seed, n, Y + 1, X + 1, salt) & mask).astype(np.int64)
    acc = (v00 * (cell - fx) * (cell - fy) + v01 * fx * (cell - fy)
           + v10 * (cell - fx) * fy + v11 * fx * fy)
    return acc >> (2 * shift)


def _crop_chunk(seed, idx, H, W, dist):
    n = idx[:, None, None].astype(np.int64)
    y = np.arange(H, dtype=np.int64)[None, :, None]
    x = np.arange(W, dtype=np.int64)[None, None, :]
    shape = (idx.shape[0], H, W)
    if dist == DIST_CONSTANT:
        return np.full(shape, 128, np.uint8), np.full(shape, 1000, np.uint16)
    if dist == DIST_NOISE:
        g = (hash5(seed, n, y, x, 8) & 255).astype(np.uint8)
        return np.broadcast_to(g, shape).copy(), np.full(shape, 1000, np.uint16)
    # --- face-like grey: 2-octave value noise, quantised to steps of 4 ---
    v16 = _value_noise(seed, n, y, x, 4, 255, 1)
    v4 = _value_noise(seed, n, y, x, 2, 63, 2)
    base = 60 + (hash5(seed, n, 0, 0, 3) % 141).astype(np.int64)
    g = base + (((v16 - 128) * 3) >> 2) + (v4 - 32)
    g = (np.clip(g, 0, 255) & ~3).astype(np.uint8)
    g = np.broadcast_to(g, shape)
    # --- depth: background plane + face ellipse with nose relief + shadow holes ---
    bg = 2000 + (hash5(seed, n, 0, 0, 4) % 1001).astype(np.int64)
    cx = W // 2 + (hash5(seed, n, 0, 0, 5) % (W // 8 + 1)).astype(np.int64) - W // 16
    cy = H // 2 + (hash5(seed, n, 0, 0, 9) % (H // 8 + 1)).astype(np.int64) - H // 16
    a = (W * 36) // 100
    b = (H * 43) // 100
    a2, b2 = a * a, b * b
    R = a2 * b2
    fd = 900 + (hash5(seed, n, 0, 0, 6) % 201).astype(np.int64)
    dx, dy = x - cx, y - cy
    e = dx * dx * b2 + dy * dy * a2
    rn = max(W // 8, 1)
    r2 = dx * dx + dy * dy
    relief = np.where(r2 < rn * rn, 40 - (40 * r2) // (rn * rn), 0)
    d = np.where(e <= R, fd - relief, bg)
    by, bx = y // 3, x // 3
    ecx, ecy = 3 * bx + 1 - cx, 3 * by + 1 - cy
    ec = ecx * ecx * b2 + ecy * ecy * a2
    near = np.abs(ec - R) * 100 < 15 * R
    p = np.where(near, 200, 10)
    hole = (hash5(seed, n, by, bx, 7) % 1000).astype(np.int64) < p
    d = np.where(hole, 0, d)
    return g.copy(), np.broadcast_to(d, shape).astype(np.uint16)


def face_crops(n: int, H: int, W: int, seed: int = 42, first_index: int = 0,
               dist: str | int = "face", chunk: int = 256):
    """Crops [n][H][W] grey u8 and depth u16 for global crop indices first_index..+n."""
    dist = DISTS[dist] if isinstance(dist, str) else int(dist)
    grey = np.empty((n, H, W), np.uint8)
    depth = np.empty((n, H, W), np.uint16)
    for s in range(0, n, chunk):
        idx = np.arange(first_index + s, first_index + min(n, s + chunk), dtype=np.int64)
        g, d = _crop_chunk(seed, idx, H, W, dist)
        grey[s:s + len(idx)] = g
        depth[s:s + len(idx)] = d
    return grey, depth


def full_rois(n: int, H: int, W: int) -> np.ndarray:
    """One ROI per image covering the whole crop: (img, 0, 0, W, H)."""
    r = np.zeros((n, 5), np.int32)
    r[:, 0] = np.arange(n)
    r[:, 3] = W
    r[:, 4] = H
    return r


def svm_weights(n_classes: int, dim: int, seed: int = 42, sigma: float = 2.0 ** -4):
    """W ~ N(0, sigma^2) fp32 [C][dim], b ~ N(0, 1) fp32 [C]; seeded, rank-independent."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x5F3]))
    W = (rng.standard_normal((n_classes, dim)) * sigma).astype(np.float32)
    b = rng.standard_normal(n_classes).astype(np.float32)
    return W, b


def random_rois(n: int, n_images: int, H: int, W: int, seed: int, min_size: int = 3,
                max_size: int | None = None, allow_outside: bool = True) -> np.ndarray:
    """Random ROI rects; with allow_outside they may stick out of the image (clamp tests)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x201]))
    max_size = max_size or max(H, W)
    w = rng.integers(min_size, max_size + 1, n)
    h = rng.integers(min_size, max_size + 1, n)
    if allow_outside:
        x = rng.integers(-4, W, n)
        y = rng.integers(-4, H, n)
    else:
        w, h = np.minimum(w, W), np.minimum(h, H)
        x = (rng.random(n) * (W - w + 1)).astype(np.int64)
        y = (rng.random(n) * (H - h + 1)).astype(np.int64)
    return np.stack([rng.integers(0, n_images, n), x, y, w, h], axis=1).astype(np.int32)


# --------------------------------------------------------------------------- GPU twin
import os as _os
import subprocess as _subprocess

_HERE = _os.path.dirname(_os.path.abspath(__file__))
_CU = _os.path.join(_HERE, "synth_gen.cu")
_SO = _os.path.join(_HERE, "libsynthgen.so")
_gpu_lib = None


def build_gpu(force: bool = False) -> str:
    """nvcc-compile synth_gen.cu for sm_100a into synthgen/libsynthgen.so (in-tree)."""
    stale = lambda: not _os.path.exists(_SO) or _os.path.getmtime(_SO) < _os.path.getmtime(_CU)
    if force or stale():
        import fcntl
        with open(_SO + ".lock", "w") as lock:  # one build among concurrent processes
            fcntl.flock(lock, fcntl.LOCK_EX)
            if force or stale():
                nvcc = _os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
                tmp = f"{_SO}.tmp{_os.getpid()}"
                _subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                                 "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-cudart",
                                 "static", "-o", tmp, _CU], check=True)
                _os.replace(tmp, _SO)
    return _SO


def gpu_face_crops(n: int, H: int, W: int, seed: int = 42, first_index: int = 0,
                   dist: str | int = "face", grey=None, depth=None, device="cuda"):
    """Same crops as face_crops(), drawn directly into CUDA tensors (torch, current stream)."""
    import ctypes

    import torch
    global _gpu_lib
    if _gpu_lib is None:
        if not _os.path.exists(_SO):
            raise ImportError(f"{_SO} missing: run __graft_entry__.build()")
        _gpu_lib = ctypes.CDLL(_SO)
        _gpu_lib.synth_face_crops.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                              ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32,
                                              ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p]
        _gpu_lib.synth_face_crops.restype = ctypes.c_int32
    dist = DISTS[dist] if isinstance(dist, str) else int(dist)
    if grey is None:
        grey = torch.empty((n, H, W), dtype=torch.uint8, device=device)
    if depth is None:
        depth = torch.empty((n, H, W), dtype=torch.uint16, device=device)
    assert grey.is_contiguous() and depth.is_contiguous() and grey.numel() == n * H * W
    st = _gpu_lib.synth_face_crops(ctypes.c_void_p(grey.data_ptr()),
                                   ctypes.c_void_p(depth.data_ptr()), n, H, W, seed & 0xFFFFFFFF,
                                   first_index, dist,
                                   ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if st != 0:
        raise RuntimeError(f"synth_face_crops failed ({st})")
    return grey, depth


# --------------------------------------------------------------------------- Kinect frame stream
def kinect_frames(n_frames: int, n_faces: int = 4, H: int = 480, W: int = 640, roi: int = 128,
                  seed: int = 42, max_step: int = 20):
    """BASELINE configs[1]: a 640x480 grey+depth frame stream with `n_faces` tracked faces.

    Face k follows a seeded straight path (<= max_step px per frame per axis, bouncing at the
    frame border, S:641's motion bound); its ROI is the roi x roi box at that position.  Grey =
    the same 2-octave value noise as face_crops() over the whole frame; depth = background
    2000..3000 mm with a face ellipse (semi-axes 0.36/0.43 roi, 900..1100 mm, nose relief) in
    every ROI.  Returns grey u8 [n][H][W], depth u16 [n][H][W], rois int32 [n*n_faces][5]."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0xF2A]))
    pos = np.stack([rng.integers(0, W - roi, n_faces), rng.integers(0, H - roi, n_faces)], 1)
    vel = rng.integers(-max_step, max_step + 1, (n_faces, 2))
    fd = rng.integers(900, 1101, n_faces)
    rois = np.zeros((n_frames * n_faces, 5), np.int32)
    grey = np.empty((n_frames, H, W), np.uint8)
    depth = np.empty((n_frames, H, W), np.uint16)
    y = np.arange(H, dtype=np.int64)[:, None]
    x = np.arange(W, dtype=np.int64)[None, :]
    a, b = (roi * 36) // 100, (roi * 43) // 100
    a2, b2 = a * a, b * b
    rn = max(roi // 8, 1)
    for f in range(n_frames):
        g, _ = face_crops(1, H, W, seed=seed, first_index=f)
        grey[f] = g[0]
        bg = 2000 + int(hash5(seed, f, 0, 0, 4) % 1001)
        d = np.full((H, W), bg, np.int64)
        for k in range(n_faces):
            for ax, lim in ((0, W - roi), (1, H - roi)):
                nxt = pos[k, ax] + vel[k, ax]
                if nxt < 0 or nxt > lim:
                    vel[k, ax] = -vel[k, ax]
                    nxt = pos[k, ax] + vel[k, ax]
                pos[k, ax] = nxt
            x0, y0 = int(pos[k, 0]), int(pos[k, 1])
            rois[f * n_faces + k] = (f, x0, y0, roi, roi)
            dx, dy = x - (x0 + roi // 2), y - (y0 + roi // 2)
            e = dx * dx * b2 + dy * dy * a2
            r2 = dx * dx + dy * dy
            relief = np.where(r2 < rn * rn, 40 - (40 * r2) // (rn * rn), 0)
            d = np.where(e <= a2 * b2, fd[k] - relief, d)
        depth[f] = d.astype(np.uint16)
    return grey, depth, rois


# --------------------------------------------------------------------------- training inputs

def train_order(n: int, epochs: int, seed: int = 42) -> np.ndarray:
    """The seeded visit order of SVM training ("samples visited in seeded-shuffle
    order"): epoch e is a permutation of 0..n-1 drawn from SeedSequence([seed, e]); the
    epochs are concatenated (int32 [epochs * n])."""
    out = np.empty(epochs * n, np.int32)
    for e in range(epochs):
        rng = np.random.default_rng(np.random.SeedSequence([seed, e, 0x5EED]))
        out[e * n:(e + 1) * n] = rng.permutation(n)
    return out
