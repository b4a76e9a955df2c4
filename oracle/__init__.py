"""CPU oracle for the fused-depth LBP + linear-SVM hot path (arXiv 1504.01883).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this
package.  The product package ``paper_1504_01883_b200`` never imports it, and
it never imports the product package: the two share no code.

The arithmetic lives in ``lbp_oracle.c`` (plain single-threaded C, citations in
its comments); this module only builds it with gcc and marshals numpy arrays
through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lbp_oracle.c")
_LIB = os.path.join(_HERE, "liblbp_oracle.so")

ORC_OK, ORC_E_ARG, ORC_E_ROI, ORC_E_GRID, ORC_E_OVERFLOW = 0, -1, -2, -3, -4
SRC_GREY, SRC_DEPTH, SRC_FUSED = 0, 1, 2

_lib = None


def build(force: bool = False) -> str:
    """Compile lbp_oracle.c into liblbp_oracle.so (gcc, -O2, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-ffp-contract=off",
               "-fno-fast-math", "-o", _LIB, _SRC]
        subprocess.run(cmd, check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64, u16, f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint16, ctypes.c_float
        L.oracle_lbp_code_window.argtypes = [P]
        L.oracle_lbp_code_window.restype = i32
        L.oracle_uniform_table.argtypes = [P]
        L.oracle_uniform_table.restype = i32
        L.oracle_lbp_map_u8.argtypes = [P, i32, i32, i64, P]
        L.oracle_lbp_map_u8.restype = i32
        L.oracle_lbp_extract.argtypes = [P, P, i32, i32, i32, i64, i64, i64, i64, P, i32,
                                         u16, u16, i32, i32, i32, P, P]
        L.oracle_lbp_extract.restype = i32
        L.oracle_lbp_extract_src.argtypes = [P, P, i32, i32, i32, i64, i64, i64, i64, P, i32,
                                             u16, u16, i32, i32, i32, i32, P, P]
        L.oracle_lbp_extract_src.restype = i32
        L.oracle_desc_pack_u8.argtypes = [P, i64, i32, i64, P, P, P, P, i32, P]
        L.oracle_desc_pack_u8.restype = i32
        L.oracle_desc_unpack_u8.argtypes = [P, i64, i32, i64, P, P, P, i32, P]
        L.oracle_desc_unpack_u8.restype = i32
        L.oracle_resize_grey.argtypes = [P, i32, i32, i64, i32, i32, P]
        L.oracle_resize_grey.restype = i32
        L.oracle_resize_depth.argtypes = [P, i32, i32, i64, i32, i32, P]
        L.oracle_resize_depth.restype = i32
        L.oracle_lbp_extract_resized.argtypes = [P, P, i32, i32, i32, i64, i64, i64, i64, P, i32,
                                                 i32, u16, u16, i32, i32, i32, i32, P, P]
        L.oracle_lbp_extract_resized.restype = i32
        L.oracle_svm_score_l1.argtypes = [P, i32, i32, i32, P, P, i32, P, P, P, f32]
        L.oracle_svm_score_l1.restype = i32
        L.oracle_svm_train_ovr.argtypes = [P, i32, i32, P, i32, P, i64, i32, P, P, P]
        L.oracle_svm_train_ovr.restype = i32
        L.oracle_svm_score.argtypes = [P, i32, i32, P, P, i32, P, P, P, f32]
        L.oracle_svm_score.restype = i32
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def lbp_code_window(window) -> int:
    """Eq. 2 on one 3x3 window (row-major, any unsigned sample width)."""
    w = np.ascontiguousarray(np.asarray(window, dtype=np.uint32).reshape(9))
    return int(lib().oracle_lbp_code_window(_ptr(w)))


def uniform_table():
    """(table[256] uint8, number of uniform codes)."""
    t = np.zeros(256, dtype=np.uint8)
    n = lib().oracle_uniform_table(_ptr(t))
    return t, int(n)


def lbp_map_u8(img: np.ndarray) -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    out = np.zeros((max(h - 2, 0), max(w - 2, 0)), dtype=np.uint8)
    st = lib().oracle_lbp_map_u8(_ptr(img), h, w, w, _ptr(out))
    if st != ORC_OK:
        raise ValueError(f"oracle_lbp_map_u8 status {st}")
    return out


def lbp_extract(grey, depth, rois, dmin: int, dmax: int,
                cells_x: int, cells_y: int, bins: int, *, source: int = SRC_GREY,
                return_status: bool = False):
    """Descriptors for ROIs of a [n_images][H][W] grey (+ optional depth) stack.

    rois: int32 [n][5] = (img, x, y, w, h).  source: SRC_GREY (codes on grey), SRC_DEPTH
    (codes on the u16 depth plane) or SRC_FUSED (grey block then depth block).  Returns
    uint16 [n][(1 or 2)*cells_y*cells_x*bins] (and int32 per-ROI status when return_status).
    """
    if grey is not None:
        grey = np.ascontiguousarray(grey, dtype=np.uint8)
        if grey.ndim == 2:
            grey = grey[None]
    if depth is not None:
        depth = np.ascontiguousarray(depth, dtype=np.uint16)
        if depth.ndim == 2:
            depth = depth[None]
        if grey is not None:
            assert depth.shape == grey.shape
    ref = grey if grey is not None else depth
    n_img, H, W = ref.shape
    rois = np.ascontiguousarray(np.asarray(rois, dtype=np.int32).reshape(-1, 5))
    n = rois.shape[0]
    dim = cells_x * cells_y * bins * (2 if source == SRC_FUSED else 1)
    desc = np.zeros((n, dim), dtype=np.uint16)
    status = np.zeros(n, dtype=np.int32)
    st = lib().oracle_lbp_extract_src(_ptr(grey), _ptr(depth), n_img, H, W, W, W, H * W, H * W,
                                      _ptr(rois), n, dmin, dmax, cells_x, cells_y, bins, source,
                                      _ptr(desc), _ptr(status))
    if st != ORC_OK:
        raise ValueError(f"oracle_lbp_extract_src status {st}")
    return (desc, status) if return_status else desc


def resize_grey(img: np.ndarray, out_h: int, out_w: int) -> np.ndarray:
    """Bilinear, half-pixel centres, round half up, exact integer arithmetic."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    out = np.zeros((out_h, out_w), np.uint8)
    st = lib().oracle_resize_grey(_ptr(img), h, w, w, out_h, out_w, _ptr(out))
    if st != ORC_OK:
        raise ValueError(f"oracle_resize_grey status {st}")
    return out


def resize_depth(img: np.ndarray, out_h: int, out_w: int) -> np.ndarray:
    """Nearest neighbour, half-pixel centres, ties toward the smaller index."""
    img = np.ascontiguousarray(img, dtype=np.uint16)
    h, w = img.shape
    out = np.zeros((out_h, out_w), np.uint16)
    st = lib().oracle_resize_depth(_ptr(img), h, w, w, out_h, out_w, _ptr(out))
    if st != ORC_OK:
        raise ValueError(f"oracle_resize_depth status {st}")
    return out


def lbp_extract_resized(grey, depth, rois, size: int, dmin: int, dmax: int, cells_x: int,
                        cells_y: int, bins: int, *, source: int = SRC_GREY,
                        return_status: bool = False):
    """Descriptors of ROIs cropped (clamped) and resized to size x size."""
    if grey is not None:
        grey = np.ascontiguousarray(grey, dtype=np.uint8)
        grey = grey[None] if grey.ndim == 2 else grey
    if depth is not None:
        depth = np.ascontiguousarray(depth, dtype=np.uint16)
        depth = depth[None] if depth.ndim == 2 else depth
    ref = grey if grey is not None else depth
    n_img, H, W = ref.shape
    rois = np.ascontiguousarray(np.asarray(rois, dtype=np.int32).reshape(-1, 5))
    n = rois.shape[0]
    dim = cells_x * cells_y * bins * (2 if source == SRC_FUSED else 1)
    desc = np.zeros((n, dim), dtype=np.uint16)
    status = np.zeros(n, dtype=np.int32)
    st = lib().oracle_lbp_extract_resized(_ptr(grey), _ptr(depth), n_img, H, W, W, W, H * W,
                                          H * W, _ptr(rois), n, size, dmin, dmax, cells_x,
                                          cells_y, bins, source, _ptr(desc), _ptr(status))
    if st != ORC_OK:
        raise ValueError(f"oracle_lbp_extract_resized status {st}")
    return (desc, status) if return_status else desc


def lbp_extract_raw(*args):
    """Direct call with the raw C argument list (for argument-validation pins)."""
    return lib().oracle_lbp_extract(*args)


def svm_score(desc: np.ndarray, W: np.ndarray, bias: np.ndarray,
              reject_threshold: float = float("-inf")):
    """Returns (scores fp32 [n][C], labels int32 [n], top fp32 [n])."""
    desc = np.ascontiguousarray(desc, dtype=np.uint16)
    W = np.ascontiguousarray(W, dtype=np.float32)
    bias = np.ascontiguousarray(bias, dtype=np.float32)
    n, dim = desc.shape
    C = W.shape[0]
    assert W.shape == (C, dim) and bias.shape == (C,)
    scores = np.zeros((n, C), dtype=np.float32)
    labels = np.zeros(n, dtype=np.int32)
    top = np.zeros(n, dtype=np.float32)
    st = lib().oracle_svm_score(_ptr(desc), n, dim, _ptr(W), _ptr(bias), C, _ptr(scores),
                                _ptr(labels), _ptr(top), reject_threshold)
    if st != ORC_OK:
        raise ValueError(f"oracle_svm_score status {st}")
    return scores, labels, top


def svm_score_l1(desc: np.ndarray, W: np.ndarray, bias: np.ndarray, block: int,
                 reject_threshold: float = float("-inf")):
    """SVM on per-block L1-normalised descriptors: (scores, labels, top)."""
    desc = np.ascontiguousarray(desc, dtype=np.uint16)
    W = np.ascontiguousarray(W, dtype=np.float32)
    bias = np.ascontiguousarray(bias, dtype=np.float32)
    n, dim = desc.shape
    C = W.shape[0]
    scores = np.zeros((n, C), dtype=np.float32)
    labels = np.zeros(n, dtype=np.int32)
    top = np.zeros(n, dtype=np.float32)
    st = lib().oracle_svm_score_l1(_ptr(desc), n, dim, block, _ptr(W), _ptr(bias), C,
                                   _ptr(scores), _ptr(labels), _ptr(top), reject_threshold)
    if st != ORC_OK:
        raise ValueError(f"oracle_svm_score_l1 status {st}")
    return scores, labels, top


def svm_train_ovr(desc: np.ndarray, labels: np.ndarray, n_classes: int, order: np.ndarray,
                  inv_lambda: int, return_z: bool = False):
    """One-vs-rest linear SVM training (exact integer Pegasos form, R20):
    (W fp32 [C][dim], bias fp32 [C]) (and the integer state z [C][dim+1])."""
    desc = np.ascontiguousarray(desc, dtype=np.uint16)
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    order = np.ascontiguousarray(order, dtype=np.int32)
    n, dim = desc.shape
    W = np.zeros((n_classes, dim), np.float32)
    b = np.zeros(n_classes, np.float32)
    z = np.zeros((n_classes, dim + 1), np.int64)
    st = lib().oracle_svm_train_ovr(_ptr(desc), n, dim, _ptr(labels), n_classes, _ptr(order),
                                    order.size, inv_lambda, _ptr(W), _ptr(b), _ptr(z))
    if st != ORC_OK:
        raise ValueError(f"oracle_svm_train_ovr status {st}")
    return (W, b, z) if return_z else (W, b)


def desc_pack_u8(desc: np.ndarray, row_base: int = 0, cap: int | None = None):
    """Descriptor compaction (R21): (packed u8 [n][dim], exceptions int64 [k][3] of
    (row, index, value) in row-major order, total exception count)."""
    desc = np.ascontiguousarray(desc, dtype=np.uint16)
    n, dim = desc.shape
    if cap is None:
        cap = int(np.count_nonzero(desc > 255))
    packed = np.zeros((n, dim), np.uint8)
    rows = np.zeros(max(cap, 1), np.int64)
    idx = np.zeros(max(cap, 1), np.int32)
    val = np.zeros(max(cap, 1), np.int32)
    cnt = np.zeros(1, np.int32)
    st = lib().oracle_desc_pack_u8(_ptr(desc), n, dim, row_base, _ptr(packed), _ptr(rows),
                                   _ptr(idx), _ptr(val), cap, _ptr(cnt))
    if st != ORC_OK:
        raise ValueError(f"oracle_desc_pack_u8 status {st}")
    k = min(int(cnt[0]), cap)
    exc = np.stack([rows[:k], idx[:k].astype(np.int64), val[:k].astype(np.int64)], 1)
    return packed, exc, int(cnt[0])


def desc_unpack_u8(packed: np.ndarray, exc: np.ndarray, row_base: int = 0) -> np.ndarray:
    """Inverse of desc_pack_u8: u16 [n][dim] from the packed rows and (row, index, value)."""
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    n, dim = packed.shape
    exc = np.asarray(exc, np.int64).reshape(-1, 3)
    rows = np.ascontiguousarray(exc[:, 0])
    idx = np.ascontiguousarray(exc[:, 1], dtype=np.int32)
    val = np.ascontiguousarray(exc[:, 2], dtype=np.int32)
    out = np.zeros((n, dim), np.uint16)
    st = lib().oracle_desc_unpack_u8(_ptr(packed), n, dim, row_base, _ptr(rows), _ptr(idx),
                                     _ptr(val), len(exc), _ptr(out))
    if st != ORC_OK:
        raise ValueError(f"oracle_desc_unpack_u8 status {st}")
    return out
