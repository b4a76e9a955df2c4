"""Thin ctypes binding of liblbpfused.so (include/lbpfused.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA library; this module only turns
torch tensors into (device pointer, geometry, stream) arguments.  There is no
CPU fallback: if the library is missing or the tensors are not on a CUDA
device, the call raises.
"""
from __future__ import annotations

import ctypes
import math
import os

import torch

from . import build as _build

LBP_OK, LBP_E_ARG, LBP_E_ROI, LBP_E_GRID, LBP_E_OVERFLOW, LBP_E_UNSUPPORTED, LBP_E_CUDA = \
    0, -1, -2, -3, -4, -5, -6
LBP_SRC_GREY, LBP_SRC_DEPTH, LBP_SRC_FUSED = 0, 1, 2
LBP_LABEL_BAD_MODEL = -2  # labels of a call whose `prepared` belongs to another model


class LbpError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {status_string(status)} ({status})")
        self.status = status


class lbp_images_t(ctypes.Structure):
    _fields_ = [("n_images", ctypes.c_int32), ("height", ctypes.c_int32),
                ("width", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("grey_pitch", ctypes.c_int64), ("depth_pitch", ctypes.c_int64),
                ("grey_img_stride", ctypes.c_int64), ("depth_img_stride", ctypes.c_int64)]


LBP_GATHER_MULTIMEM, LBP_GATHER_PEERS, LBP_GATHER_MAX_DST = 1, 2, 8


class lbp_gather_dst_t(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("n_dst", ctypes.c_int32),
                ("base", ctypes.c_uint64 * LBP_GATHER_MAX_DST),
                ("desc_offset", ctypes.c_int64), ("desc_pitch", ctypes.c_int64),
                ("labels_offset", ctypes.c_int64), ("row_base", ctypes.c_int64)]


_lib = None


def lib():
    """Load liblbpfused.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(_build.LIB):
            raise ImportError(f"{_build.LIB} is missing: run `python __graft_entry__.py build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(_build.LIB)
        P, i32, u16, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint16, ctypes.c_float
        sz = ctypes.c_size_t
        L.lbp_descriptor_dim.argtypes = [i32, i32, i32]
        L.lbp_descriptor_dim.restype = i32
        L.lbp_status_string.argtypes = [i32]
        L.lbp_status_string.restype = ctypes.c_char_p
        L.lbp_fused_extract.argtypes = [P, P, lbp_images_t, P, i32, u16, u16, i32, i32, i32, P, P, P]
        L.lbp_fused_extract.restype = i32
        L.lbp_extract_source.argtypes = [P, P, lbp_images_t, P, i32, u16, u16, i32, i32, i32, i32,
                                         P, P, P]
        L.lbp_extract_source.restype = i32
        L.lbp_extract_resized.argtypes = [P, P, lbp_images_t, P, i32, i32, u16, u16, i32, i32,
                                          i32, i32, P, P, P]
        L.lbp_extract_resized.restype = i32
        L.lbp_recognize.argtypes = [P, P, lbp_images_t, P, i32, u16, u16, i32, i32, i32, P, P,
                                    i32, P, sz, f32, P, P, P, P, P, P]
        L.lbp_recognize.restype = i32
        L.svm_score.argtypes = [P, i32, i32, P, P, i32, P, sz, P, P, P, f32, P]
        L.svm_score.restype = i32
        L.svm_score_l1.argtypes = [P, i32, i32, i32, P, P, i32, P, P, P, f32, P]
        L.svm_score_l1.restype = i32
        L.svm_train_ovr.argtypes = [P, i32, i32, P, i32, P, ctypes.c_int64, i32, P, P, P, P]
        L.svm_train_ovr.restype = i32
        i64 = ctypes.c_int64
        L.lbp_desc_pack_u8.argtypes = [P, i64, i32, i64, P, P, i32, P, P]
        L.lbp_desc_pack_u8.restype = i32
        L.lbp_desc_unpack_u8.argtypes = [P, i64, i32, i64, P, P, i32, i32, P, P]
        L.lbp_desc_unpack_u8.restype = i32
        L.lbp_extract_gather.argtypes = [P, P, lbp_images_t, P, i32, u16, u16, i32, i32, i32, P,
                                         lbp_gather_dst_t, P, P, P]
        L.lbp_extract_gather.restype = i32
        L.lbp_u8_exc_cap_min.argtypes = [lbp_images_t, i32]
        L.lbp_u8_exc_cap_min.restype = i32
        L.lbp_extract_u8.argtypes = [P, P, lbp_images_t, P, i32, u16, u16, i32, i32, i32, P, i64,
                                     P, P, i32, P, P, P]
        L.lbp_extract_u8.restype = i32
        L.svm_workspace_u8_bytes.argtypes = [i32, i32]
        L.svm_workspace_u8_bytes.restype = sz
        L.svm_prepare_u8.argtypes = [P, i32, i32, P, sz, P]
        L.svm_prepare_u8.restype = i32
        L.svm_score_u8.argtypes = [P, i64, P, P, i32, i32, i32, P, P, i32, P, sz, P, P, P, f32, P]
        L.svm_score_u8.restype = i32
        L.svm_workspace_bytes.argtypes = [i32, i32]
        L.svm_workspace_bytes.restype = sz
        L.svm_prepare.argtypes = [P, i32, i32, P, sz, P]
        L.svm_prepare.restype = i32
        L.lbp_recognize_workspace_bytes.argtypes = [lbp_images_t, i32, i32, i32, i32, i32]
        L.lbp_recognize_workspace_bytes.restype = sz
        L.lbp_recognize_host.argtypes = [P, P, lbp_images_t, P, i32, u16, u16, i32, i32, i32,
                                         P, P, i32, P, sz, f32, P, sz, P, P, P]
        L.lbp_recognize_host.restype = i32
        _lib = L
    return _lib


def status_string(status: int) -> str:
    return lib().lbp_status_string(int(status)).decode()


def lbp_descriptor_dim(cells_x: int, cells_y: int, bins: int) -> int:
    d = lib().lbp_descriptor_dim(cells_x, cells_y, bins)
    if d < 0:
        raise LbpError(d, "lbp_descriptor_dim")
    return d


def _require(ok: bool, what: str) -> None:
    """Argument check that survives `python -O` (the C ABI trusts these sizes and types)."""
    if not ok:
        raise ValueError(f"lbpfused: argument check failed: {what}")


def _out(t, dtype, n, what: str, device=None) -> None:
    """A caller-provided output (or input) buffer: dtype, contiguous, >= n elements, and on
    `device` when given (the C ABI writes n elements through the raw pointer)."""
    if t is None:
        return
    _require(t.dtype == dtype, f"{what}.dtype == {dtype}")
    _require(t.is_contiguous(), f"{what}.is_contiguous()")
    _require(t.numel() >= n, f"{what}.numel() >= {n}")
    if device is not None:
        _require(t.device == device, f"{what}.device == {device}")


def _model(W, bias, dim, device, what):
    """W fp32 [C][dim] contiguous and bias fp32 [C] contiguous on `device`."""
    _require(W.dtype == torch.float32 and W.is_contiguous() and W.dim() == 2,
             f"{what}: W fp32 contiguous [C][dim]")
    C = W.shape[0]
    if W.shape[1] != dim or bias.numel() != C:
        raise LbpError(LBP_E_ARG, f"{what}: weight shape mismatch")
    _out(bias, torch.float32, C, "bias", device)
    _require(W.device == device, f"W.device == {device}")
    return C


def _prepared(prepared, C, dim, device):
    """svm_prepare() workspace: uint8 on the device, at least svm_workspace_bytes(C, dim)."""
    if prepared is None:
        return 0
    _require(prepared.dtype == torch.uint8 and prepared.is_contiguous(),
             "prepared.dtype == torch.uint8 and prepared.is_contiguous()")
    _require(prepared.device == device, f"prepared.device == {device}")
    _require(prepared.numel() >= svm_workspace_bytes(C, dim),
             "prepared.numel() >= svm_workspace_bytes(C, dim)")
    return prepared.numel()


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _stack3(t: torch.Tensor) -> torch.Tensor:
    return t.unsqueeze(0) if t.dim() == 2 else t


def images_geometry(grey: torch.Tensor | None, depth: torch.Tensor | None) -> lbp_images_t:
    """lbp_images_t from [n_images][H][W] (or [H][W]) tensors with unit column stride."""
    if grey is None:  # depth-only stack (LBP_SRC_DEPTH)
        d = _stack3(depth)
        if d.stride(2) != 1:
            raise ValueError("depth rows must be contiguous")
        n, H, W = d.shape
        return lbp_images_t(n, H, W, 0, W, d.stride(1), n * H * W, d.stride(0))
    g = _stack3(grey)
    if g.stride(2) != 1:
        raise ValueError("grey rows must be contiguous")
    n, H, W = g.shape
    geom = lbp_images_t(n, H, W, 0, g.stride(1), g.stride(1), g.stride(0), g.stride(0))
    if depth is not None:
        d = _stack3(depth)
        if tuple(d.shape) != (n, H, W) or d.stride(2) != 1:
            raise ValueError("depth must match grey's shape with contiguous rows")
        geom.depth_pitch, geom.depth_img_stride = d.stride(1), d.stride(0)
    return geom


def _check_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("lbpfused operates on CUDA tensors only (no CPU fallback)")


def lbp_fused_extract(grey: torch.Tensor, depth: torch.Tensor | None, rois: torch.Tensor,
                      dmin: int, dmax: int, cells_x: int, cells_y: int, bins: int,
                      out: torch.Tensor | None = None, roi_status: torch.Tensor | None = None,
                      stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Descriptors u16 [n_rois][cells_y*cells_x*bins] of the ROIs (int32 [n][5] = img,x,y,w,h)."""
    _check_cuda(grey, depth, rois, out, roi_status)
    _require(grey.dtype == torch.uint8 and (depth is None or depth.dtype == torch.uint16),
             "grey.dtype == torch.uint8 and (depth is None or depth.dtype == torch.uint16)")
    _require(rois.dtype == torch.int32 and rois.is_contiguous() and rois.shape[-1] == 5,
             "rois.dtype == torch.int32 and rois.is_contiguous() and rois.shape[-1] == 5")
    n = rois.shape[0]
    dim = lbp_descriptor_dim(cells_x, cells_y, bins)
    if out is None:
        out = torch.empty((n, dim), dtype=torch.uint16, device=grey.device)
    _require(out.dtype == torch.uint16 and out.is_contiguous() and out.numel() >= n * dim,
             "out.dtype == torch.uint16 and out.is_contiguous() and out.numel() >= n * dim")
    if roi_status is not None:
        _require(roi_status.dtype == torch.int32 and roi_status.numel() >= n,
                 "roi_status.dtype == torch.int32 and roi_status.numel() >= n")
    st = lib().lbp_fused_extract(_ptr(grey), _ptr(depth), images_geometry(grey, depth),
                                 _ptr(rois), n, dmin, dmax, cells_x, cells_y, bins, _ptr(out),
                                 _ptr(roi_status), _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "lbp_fused_extract")
    return out


def lbp_extract_source(grey: torch.Tensor | None, depth: torch.Tensor | None,
                       rois: torch.Tensor, dmin: int, dmax: int, cells_x: int, cells_y: int,
                       bins: int, source: int, out: torch.Tensor | None = None,
                       roi_status: torch.Tensor | None = None,
                       stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Descriptors with the code source selectable (LBP_SRC_GREY / _DEPTH / _FUSED): u16
    [n_rois][dim] (grey or depth) or [n_rois][2*dim] (fused: grey block then depth block)."""
    _check_cuda(grey, depth, rois, out, roi_status)
    _require(grey is None or grey.dtype == torch.uint8, "grey is None or grey.dtype == torch.uint8")
    _require(depth is None or depth.dtype == torch.uint16,
             "depth is None or depth.dtype == torch.uint16")
    _require(rois.dtype == torch.int32 and rois.is_contiguous() and rois.shape[-1] == 5,
             "rois.dtype == torch.int32 and rois.is_contiguous() and rois.shape[-1] == 5")
    if grey is None and depth is None:
        raise LbpError(LBP_E_ARG, "lbp_extract_source: no image plane")
    n = rois.shape[0]
    dim = lbp_descriptor_dim(cells_x, cells_y, bins) * (2 if source == LBP_SRC_FUSED else 1)
    dev = (grey if grey is not None else depth).device
    if out is None:
        out = torch.empty((n, dim), dtype=torch.uint16, device=dev)
    _require(out.dtype == torch.uint16 and out.is_contiguous() and out.numel() >= n * dim,
             "out.dtype == torch.uint16 and out.is_contiguous() and out.numel() >= n * dim")
    if roi_status is not None:
        _require(roi_status.dtype == torch.int32 and roi_status.numel() >= n,
                 "roi_status.dtype == torch.int32 and roi_status.numel() >= n")
    st = lib().lbp_extract_source(_ptr(grey), _ptr(depth), images_geometry(grey, depth),
                                  _ptr(rois), n, dmin, dmax, cells_x, cells_y, bins, source,
                                  _ptr(out), _ptr(roi_status), _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "lbp_extract_source")
    return out


def gather_dst(mode: int, bases, desc_offset: int, desc_pitch: int, labels_offset: int,
               row_base: int) -> lbp_gather_dst_t:
    """lbp_gather_dst_t from plain integers (device addresses of the destinations)."""
    bases = [int(b) for b in bases]
    if not 1 <= len(bases) <= LBP_GATHER_MAX_DST:
        raise ValueError("gather: 1..8 destinations")
    arr = (ctypes.c_uint64 * LBP_GATHER_MAX_DST)(*(bases + [0] * (LBP_GATHER_MAX_DST - len(bases))))
    return lbp_gather_dst_t(mode, len(bases), arr, desc_offset, desc_pitch, labels_offset,
                            row_base)


def lbp_extract_gather(grey: torch.Tensor, depth: torch.Tensor | None, rois: torch.Tensor,
                       dmin: int, dmax: int, cells_x: int, cells_y: int, bins: int,
                       labels: torch.Tensor | None, dst: lbp_gather_dst_t,
                       scratch: torch.Tensor | None = None,
                       roi_status: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Fused database build step (include/lbpfused.h lbp_extract_gather): descriptors of the
    ROIs written by the extraction epilogue into every destination of `dst` (multicast or peer
    addresses).  Returns the local scratch (rows of ROIs off the fast path live there)."""
    _check_cuda(grey, depth, rois, labels, scratch, roi_status)
    _require(grey.dtype == torch.uint8 and (depth is None or depth.dtype == torch.uint16),
             "grey.dtype == torch.uint8 and (depth is None or depth.dtype == torch.uint16)")
    _require(rois.dtype == torch.int32 and rois.is_contiguous() and rois.shape[-1] == 5,
             "rois.dtype == torch.int32 and rois.is_contiguous() and rois.shape[-1] == 5")
    n = rois.shape[0]
    dim = lbp_descriptor_dim(cells_x, cells_y, bins)
    dev = grey.device
    if scratch is None:
        scratch = torch.empty((n, dim), dtype=torch.uint16, device=dev)
    _out(scratch, torch.uint16, n * dim, "scratch", dev)
    _out(labels, torch.int32, n, "labels", dev)
    _out(roi_status, torch.int32, n, "roi_status", dev)
    st = lib().lbp_extract_gather(_ptr(grey), _ptr(depth), images_geometry(grey, depth),
                                  _ptr(rois), n, dmin, dmax, cells_x, cells_y, bins,
                                  _ptr(labels), dst, _ptr(scratch), _ptr(roi_status),
                                  _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "lbp_extract_gather")
    return scratch


def lbp_extract_resized(grey: torch.Tensor | None, depth: torch.Tensor | None,
                        rois: torch.Tensor, size: int, dmin: int, dmax: int, cells_x: int,
                        cells_y: int, bins: int, source: int = LBP_SRC_GREY,
                        out: torch.Tensor | None = None,
                        roi_status: torch.Tensor | None = None,
                        stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Descriptors of the ROIs cropped (clamped) and resized to size x size on the GPU
    (grey bilinear, depth nearest)."""
    _check_cuda(grey, depth, rois, out, roi_status)
    _require(grey is None or grey.dtype == torch.uint8, "grey is None or grey.dtype == torch.uint8")
    _require(depth is None or depth.dtype == torch.uint16,
             "depth is None or depth.dtype == torch.uint16")
    _require(rois.dtype == torch.int32 and rois.is_contiguous() and rois.shape[-1] == 5,
             "rois.dtype == torch.int32 and rois.is_contiguous() and rois.shape[-1] == 5")
    if grey is None and depth is None:
        raise LbpError(LBP_E_ARG, "lbp_extract_resized: no image plane")
    n = rois.shape[0]
    dim = lbp_descriptor_dim(cells_x, cells_y, bins) * (2 if source == LBP_SRC_FUSED else 1)
    dev = (grey if grey is not None else depth).device
    if out is None:
        out = torch.empty((n, dim), dtype=torch.uint16, device=dev)
    _require(out.dtype == torch.uint16 and out.is_contiguous() and out.numel() >= n * dim,
             "out.dtype == torch.uint16 and out.is_contiguous() and out.numel() >= n * dim")
    if roi_status is not None:
        _require(roi_status.dtype == torch.int32 and roi_status.numel() >= n,
                 "roi_status.dtype == torch.int32 and roi_status.numel() >= n")
    st = lib().lbp_extract_resized(_ptr(grey), _ptr(depth), images_geometry(grey, depth),
                                   _ptr(rois), n, size, dmin, dmax, cells_x, cells_y, bins,
                                   source, _ptr(out), _ptr(roi_status), _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "lbp_extract_resized")
    return out


def lbp_recognize(grey: torch.Tensor, depth: torch.Tensor | None, rois: torch.Tensor,
                  dmin: int, dmax: int, cells_x: int, cells_y: int, bins: int, W: torch.Tensor,
                  bias: torch.Tensor, prepared=None, reject_threshold: float = -math.inf,
                  want_scores: bool = False, desc: torch.Tensor | None = None,
                  labels: torch.Tensor | None = None, top_score: torch.Tensor | None = None,
                  roi_status: torch.Tensor | None = None,
                  stream: torch.cuda.Stream | None = None):
    """Descriptors + SVM in one call (one fused launch for small batches):
    returns (desc u16 [n][dim], scores fp32 [n][C] or None, labels int32 [n], top fp32 [n])."""
    _check_cuda(grey, depth, rois, W, bias, prepared, desc, labels, top_score, roi_status)
    _require(grey.dtype == torch.uint8 and (depth is None or depth.dtype == torch.uint16),
             "grey.dtype == torch.uint8 and (depth is None or depth.dtype == torch.uint16)")
    _require(rois.dtype == torch.int32 and rois.is_contiguous() and rois.shape[-1] == 5,
             "rois.dtype == torch.int32 and rois.is_contiguous() and rois.shape[-1] == 5")
    n = rois.shape[0]
    dim = lbp_descriptor_dim(cells_x, cells_y, bins)
    dev = grey.device
    C = _model(W, bias, dim, dev, "lbp_recognize")
    pbytes = _prepared(prepared, C, dim, dev)
    if desc is None:
        desc = torch.empty((n, dim), dtype=torch.uint16, device=dev)
    if labels is None:
        labels = torch.empty(n, dtype=torch.int32, device=dev)
    if top_score is None:
        top_score = torch.empty(n, dtype=torch.float32, device=dev)
    _out(desc, torch.uint16, n * dim, "desc", dev)
    _out(labels, torch.int32, n, "labels", dev)
    _out(top_score, torch.float32, n, "top_score", dev)
    _out(roi_status, torch.int32, n, "roi_status", dev)
    _require(rois.device == dev and (depth is None or depth.device == dev),
             "rois and depth on grey's device")
    scores = torch.empty((n, C), dtype=torch.float32, device=dev) if want_scores else None
    st = lib().lbp_recognize(_ptr(grey), _ptr(depth), images_geometry(grey, depth), _ptr(rois),
                             n, dmin, dmax, cells_x, cells_y, bins, _ptr(W), _ptr(bias), C,
                             _ptr(prepared), pbytes, reject_threshold, _ptr(desc),
                             _ptr(roi_status), _ptr(scores), _ptr(labels), _ptr(top_score),
                             _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "lbp_recognize")
    return desc, scores, labels, top_score


def svm_workspace_bytes(n_classes: int, dim: int) -> int:
    return int(lib().svm_workspace_bytes(n_classes, dim))


def svm_prepare(W: torch.Tensor, stream=None) -> torch.Tensor | None:
    """Digit-plane workspace for the tensor-core scorer, or None when that path does not apply."""
    _check_cuda(W)
    C, dim = W.shape
    nbytes = svm_workspace_bytes(C, dim)
    if nbytes == 0:
        return None
    ws = torch.empty(nbytes, dtype=torch.uint8, device=W.device)
    st = lib().svm_prepare(_ptr(W), C, dim, _ptr(ws), nbytes, _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "svm_prepare")
    return ws


def svm_score(desc: torch.Tensor, W: torch.Tensor, bias: torch.Tensor, prepared=None,
              reject_threshold: float = -math.inf, want_scores: bool = True,
              labels: torch.Tensor | None = None, top_score: torch.Tensor | None = None,
              scores: torch.Tensor | None = None, stream=None):
    """(scores fp32 [n][C] or None, labels int32 [n], top fp32 [n]) of the linear OvR SVM."""
    _check_cuda(desc, W, bias, prepared)
    _require(desc.dtype == torch.uint16 and desc.is_contiguous() and desc.dim() == 2,
             "desc.dtype == torch.uint16 and desc.is_contiguous() and desc.dim() == 2")
    n, dim = desc.shape
    dev = desc.device
    C = _model(W, bias, dim, dev, "svm_score")
    pbytes = _prepared(prepared, C, dim, dev)
    if want_scores and scores is None:
        scores = torch.empty((n, C), dtype=torch.float32, device=dev)
    if labels is None:
        labels = torch.empty(n, dtype=torch.int32, device=dev)
    if top_score is None:
        top_score = torch.empty(n, dtype=torch.float32, device=dev)
    _out(labels, torch.int32, n, "labels", dev)
    _out(top_score, torch.float32, n, "top_score", dev)
    if want_scores:
        _out(scores, torch.float32, n * C, "scores", dev)
    st = lib().svm_score(_ptr(desc), n, dim, _ptr(W), _ptr(bias), C, _ptr(prepared), pbytes,
                         _ptr(scores if want_scores else None), _ptr(labels), _ptr(top_score),
                         reject_threshold, _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "svm_score")
    return (scores if want_scores else None), labels, top_score


# ---- compact descriptors (include/lbpfused.h lbp_extract_u8 / svm_score_u8)

class CompactDesc:
    """The compact descriptor of lbp_extract_u8: packed u8 [n][dim] = count & 255 (low byte),
    exc_n int32 [n], exc int32 [n][cap] holding the uint32 records (d << 16) | count of the
    entries above 255 (the first exc_n[i] of row i)."""

    def __init__(self, packed: torch.Tensor, exc_n: torch.Tensor, exc: torch.Tensor):
        self.packed, self.exc_n, self.exc = packed, exc_n, exc

    @property
    def n(self) -> int:
        return self.packed.shape[0]

    @property
    def dim(self) -> int:
        return self.packed.shape[1]

    @property
    def cap(self) -> int:
        return self.exc.shape[1]

    @staticmethod
    def empty(n: int, dim: int, cap: int, device) -> "CompactDesc":
        return CompactDesc(torch.empty((n, dim), dtype=torch.uint8, device=device),
                           torch.empty(n, dtype=torch.int32, device=device),
                           torch.empty((n, max(cap, 1)), dtype=torch.int32, device=device))

    def _check(self, n: int, dim: int, device) -> None:
        _out(self.packed, torch.uint8, n * dim, "packed", device)
        _require(self.packed.dim() == 2 and self.packed.shape[1] == dim,
                 f"packed is [n][{dim}]")
        _out(self.exc_n, torch.int32, n, "exc_n", device)
        _require(self.exc.dtype == torch.int32 and self.exc.is_contiguous() and
                 self.exc.dim() == 2 and self.exc.shape[0] >= n, "exc int32 [n][cap]")
        _require(self.exc.device == device, f"exc.device == {device}")


def lbp_u8_exc_cap_min(geom: lbp_images_t, dim: int) -> int:
    v = lib().lbp_u8_exc_cap_min(geom, dim)
    if v < 0:
        raise LbpError(v, "lbp_u8_exc_cap_min")
    return v


def lbp_extract_u8(grey: torch.Tensor, depth: torch.Tensor | None, rois: torch.Tensor,
                   dmin: int, dmax: int, cells_x: int, cells_y: int, bins: int,
                   out: CompactDesc | None = None, cap: int | None = None,
                   scratch: torch.Tensor | None = None, roi_status: torch.Tensor | None = None,
                   stream=None) -> CompactDesc:
    """Compact descriptors (CompactDesc) of the ROIs: lbp_fused_extract's rows as u8 + records
    of the entries above 255, written by the extraction kernel's epilogue."""
    _check_cuda(grey, depth, rois, scratch, roi_status)
    _require(grey.dtype == torch.uint8 and (depth is None or depth.dtype == torch.uint16),
             "grey.dtype == torch.uint8 and (depth is None or depth.dtype == torch.uint16)")
    _require(rois.dtype == torch.int32 and rois.is_contiguous() and rois.shape[-1] == 5,
             "rois.dtype == torch.int32 and rois.is_contiguous() and rois.shape[-1] == 5")
    n = rois.shape[0]
    dim = lbp_descriptor_dim(cells_x, cells_y, bins)
    geom = images_geometry(grey, depth)
    dev = grey.device
    if out is None:
        out = CompactDesc.empty(n, dim, cap if cap is not None else lbp_u8_exc_cap_min(geom, dim),
                                dev)
    out._check(n, dim, dev)
    _out(scratch, torch.uint16, n * dim, "scratch", dev)
    _out(roi_status, torch.int32, n, "roi_status", dev)
    st = lib().lbp_extract_u8(_ptr(grey), _ptr(depth), geom, _ptr(rois), n, dmin, dmax,
                              cells_x, cells_y, bins, _ptr(out.packed), dim, _ptr(out.exc_n),
                              _ptr(out.exc), out.cap, _ptr(scratch), _ptr(roi_status),
                              _stream(stream))
    if st == LBP_E_ARG and scratch is None and n > 0:
        # off the TMA kernel (small batch / other geometry): extract + pack via a u16 scratch
        scratch = torch.empty((n, dim), dtype=torch.uint16, device=dev)
        st = lib().lbp_extract_u8(_ptr(grey), _ptr(depth), geom, _ptr(rois), n, dmin, dmax,
                                  cells_x, cells_y, bins, _ptr(out.packed), dim,
                                  _ptr(out.exc_n), _ptr(out.exc), out.cap, _ptr(scratch),
                                  _ptr(roi_status), _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "lbp_extract_u8")
    return out


def svm_workspace_u8_bytes(n_classes: int, dim: int) -> int:
    return int(lib().svm_workspace_u8_bytes(n_classes, dim))


def svm_prepare_u8(W: torch.Tensor, stream=None) -> torch.Tensor | None:
    """Digit-plane workspace of svm_score_u8's tensor-core path (None if it does not apply)."""
    _check_cuda(W)
    _require(W.dtype == torch.float32 and W.is_contiguous() and W.dim() == 2,
             "W fp32 contiguous [C][dim]")
    C, dim = W.shape
    nbytes = svm_workspace_u8_bytes(C, dim)
    if nbytes == 0:
        return None
    ws = torch.empty(nbytes, dtype=torch.uint8, device=W.device)
    st = lib().svm_prepare_u8(_ptr(W), C, dim, _ptr(ws), nbytes, _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "svm_prepare_u8")
    return ws


def svm_score_u8(cd: CompactDesc, W: torch.Tensor, bias: torch.Tensor, prepared=None,
                 reject_threshold: float = -math.inf, want_scores: bool = True,
                 labels: torch.Tensor | None = None, top_score: torch.Tensor | None = None,
                 scores: torch.Tensor | None = None, stream=None):
    """svm_score on a CompactDesc: (scores or None, labels, top)."""
    _check_cuda(W, bias, prepared)
    n, dim = cd.n, cd.dim
    dev = cd.packed.device
    cd._check(n, dim, dev)
    C = _model(W, bias, dim, dev, "svm_score_u8")
    pbytes = 0
    if prepared is not None:
        _require(prepared.dtype == torch.uint8 and prepared.is_contiguous() and
                 prepared.device == dev, "prepared uint8 contiguous on the descriptors' device")
        _require(prepared.numel() >= svm_workspace_u8_bytes(C, dim),
                 "prepared.numel() >= svm_workspace_u8_bytes(C, dim)")
        pbytes = prepared.numel()
    if want_scores and scores is None:
        scores = torch.empty((n, C), dtype=torch.float32, device=dev)
    if labels is None:
        labels = torch.empty(n, dtype=torch.int32, device=dev)
    if top_score is None:
        top_score = torch.empty(n, dtype=torch.float32, device=dev)
    _out(labels, torch.int32, n, "labels", dev)
    _out(top_score, torch.float32, n, "top_score", dev)
    if want_scores:
        _out(scores, torch.float32, n * C, "scores", dev)
    st = lib().svm_score_u8(_ptr(cd.packed), dim, _ptr(cd.exc_n), _ptr(cd.exc), cd.cap, n, dim,
                            _ptr(W), _ptr(bias), C, _ptr(prepared), pbytes,
                            _ptr(scores if want_scores else None), _ptr(labels),
                            _ptr(top_score), reject_threshold, _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "svm_score_u8")
    return (scores if want_scores else None), labels, top_score


def lbp_recognize_workspace_bytes(geom: lbp_images_t, has_depth: bool, n_rois: int,
                                  cells_x: int, cells_y: int, bins: int) -> int:
    return int(lib().lbp_recognize_workspace_bytes(geom, int(has_depth), n_rois, cells_x,
                                                   cells_y, bins))


def lbp_recognize_host(grey_h: torch.Tensor, depth_h: torch.Tensor | None, rois_h: torch.Tensor,
                       dmin: int, dmax: int, cells_x: int, cells_y: int, bins: int,
                       W: torch.Tensor, bias: torch.Tensor, prepared, workspace: torch.Tensor,
                       labels_h: torch.Tensor, top_h: torch.Tensor,
                       reject_threshold: float = -math.inf, stream=None) -> None:
    """End-to-end call from (pinned) HOST tensors; results land in labels_h / top_h after a
    sync of `stream`."""
    _check_cuda(W, bias, workspace, prepared)
    for t in (grey_h, depth_h, rois_h, labels_h, top_h):
        if t is not None and t.is_cuda:
            raise ValueError("lbp_recognize_host takes host tensors")
    _require(grey_h.dtype == torch.uint8 and (depth_h is None or depth_h.dtype == torch.uint16),
             "grey_h u8 and depth_h u16")
    _require(rois_h.dtype == torch.int32 and rois_h.is_contiguous() and rois_h.shape[-1] == 5,
             "rois_h.dtype == torch.int32 and rois_h.is_contiguous() and rois_h.shape[-1] == 5")
    _require(workspace.dtype == torch.uint8 and workspace.is_contiguous(),
             "workspace.dtype == torch.uint8 and workspace.is_contiguous()")
    geom = images_geometry(grey_h, depth_h)
    n = rois_h.shape[0]
    dim = lbp_descriptor_dim(cells_x, cells_y, bins)
    C = _model(W, bias, dim, W.device, "lbp_recognize_host")
    pbytes = _prepared(prepared, C, dim, W.device)
    _out(labels_h, torch.int32, n, "labels_h")
    _out(top_h, torch.float32, n, "top_h")
    st = lib().lbp_recognize_host(_ptr(grey_h), _ptr(depth_h), geom, _ptr(rois_h), n, dmin, dmax,
                                  cells_x, cells_y, bins, _ptr(W), _ptr(bias), C,
                                  _ptr(prepared), pbytes, reject_threshold, _ptr(workspace),
                                  workspace.numel(), _ptr(labels_h), _ptr(top_h), _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "lbp_recognize_host")


def svm_score_l1(desc: torch.Tensor, W: torch.Tensor, bias: torch.Tensor, block: int,
                 reject_threshold: float = -math.inf, want_scores: bool = True,
                 stream=None):
    """(scores or None, labels, top) of the SVM on per-block L1-normalised descriptors."""
    _check_cuda(desc, W, bias)
    _require(desc.dtype == torch.uint16 and desc.is_contiguous(),
             "desc.dtype == torch.uint16 and desc.is_contiguous()")
    _require(W.dtype == torch.float32 and W.is_contiguous() and bias.dtype == torch.float32,
             "W.dtype == torch.float32 and W.is_contiguous() and bias.dtype == torch.float32")
    n, dim = desc.shape
    C = W.shape[0]
    if W.shape[1] != dim or bias.numel() != C:
        raise LbpError(LBP_E_ARG, "svm_score_l1: dimension mismatch")
    dev = desc.device
    scores = torch.empty((n, C), dtype=torch.float32, device=dev) if want_scores else None
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    top = torch.empty(n, dtype=torch.float32, device=dev)
    st = lib().svm_score_l1(_ptr(desc), n, dim, block, _ptr(W), _ptr(bias), C, _ptr(scores),
                            _ptr(labels), _ptr(top), reject_threshold, _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "svm_score_l1")
    return scores, labels, top


def svm_train_ovr(desc: torch.Tensor, labels: torch.Tensor, n_classes: int, order: torch.Tensor,
                  inv_lambda: int, return_z: bool = False, stream=None):
    """One-vs-rest linear SVM training on the GPU (exact integer Pegasos form): returns
    (W fp32 [C][dim], bias fp32 [C]) (and z int64 [C][dim+1] when return_z)."""
    _check_cuda(desc, labels, order)
    _require(desc.dtype == torch.uint16 and desc.is_contiguous(),
             "desc.dtype == torch.uint16 and desc.is_contiguous()")
    _require(labels.dtype == torch.int32 and order.dtype == torch.int32 and order.is_contiguous(),
             "labels.dtype == torch.int32 and order.dtype == torch.int32 and order.is_contiguous()")
    n, dim = desc.shape
    dev = desc.device
    W = torch.empty((n_classes, dim), dtype=torch.float32, device=dev)
    b = torch.empty(n_classes, dtype=torch.float32, device=dev)
    z = torch.empty((n_classes, dim + 1), dtype=torch.int64, device=dev) if return_z else None
    st = lib().svm_train_ovr(_ptr(desc), n, dim, _ptr(labels), n_classes, _ptr(order),
                             order.numel(), inv_lambda, _ptr(W), _ptr(b), _ptr(z),
                             _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "svm_train_ovr")
    return (W, b, z) if return_z else (W, b)


def desc_pack_u8(desc: torch.Tensor, row_base: int = 0, cap: int = 4096,
                 packed: torch.Tensor | None = None, exc: torch.Tensor | None = None,
                 count: torch.Tensor | None = None, stream=None):
    """Descriptor compaction (lbp_desc_pack_u8): returns (packed u8 [n][dim], exceptions int32
    [cap][4] = lbp_desc_exc_t records (row lo, row hi, index, value), count int32 [1]).
    count > cap after the stream synchronises means the list was truncated."""
    _check_cuda(desc, packed, exc, count)
    _require(desc.dtype == torch.uint16 and desc.is_contiguous() and desc.dim() == 2,
             "desc.dtype == torch.uint16 and desc.is_contiguous() and desc.dim() == 2")
    n, dim = desc.shape
    dev = desc.device
    if packed is None:
        packed = torch.empty((n, dim), dtype=torch.uint8, device=dev)
    if exc is None:
        exc = torch.empty((max(cap, 1), 4), dtype=torch.int32, device=dev)
    if count is None:
        count = torch.empty(1, dtype=torch.int32, device=dev)
    _require(packed.dtype == torch.uint8 and packed.is_contiguous() and packed.numel() >= n * dim,
             "packed.dtype == torch.uint8 and packed.is_contiguous() and packed.numel() >= n * dim")
    _require(exc.dtype == torch.int32 and exc.is_contiguous() and exc.numel() >= 4 * cap,
             "exc.dtype == torch.int32 and exc.is_contiguous() and exc.numel() >= 4 * cap")
    st = lib().lbp_desc_pack_u8(_ptr(desc), n, dim, row_base, _ptr(packed), _ptr(exc), cap,
                                _ptr(count), _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "lbp_desc_pack_u8")
    return packed, exc, count


def desc_unpack_u8(packed: torch.Tensor, exc: torch.Tensor, counts: torch.Tensor, cap: int,
                   row_base: int = 0, out: torch.Tensor | None = None, stream=None):
    """Inverse of desc_pack_u8 (lbp_desc_unpack_u8): u16 [n][dim] from packed u8 [n][dim] and
    len(counts) exception lists of `cap` records each (exc int32 [len(counts) * cap][4])."""
    _check_cuda(packed, exc, counts, out)
    _require(packed.dtype == torch.uint8 and packed.is_contiguous() and packed.dim() == 2,
             "packed.dtype == torch.uint8 and packed.is_contiguous() and packed.dim() == 2")
    _require(exc.dtype == torch.int32 and exc.is_contiguous(),
             "exc.dtype == torch.int32 and exc.is_contiguous()")
    _require(counts.dtype == torch.int32 and counts.is_contiguous(),
             "counts.dtype == torch.int32 and counts.is_contiguous()")
    n, dim = packed.shape
    n_lists = counts.numel()
    _require(exc.numel() >= 4 * n_lists * cap, "exc.numel() >= 4 * n_lists * cap")
    if out is None:
        out = torch.empty((n, dim), dtype=torch.uint16, device=packed.device)
    _require(out.dtype == torch.uint16 and out.is_contiguous() and out.numel() >= n * dim,
             "out.dtype == torch.uint16 and out.is_contiguous() and out.numel() >= n * dim")
    st = lib().lbp_desc_unpack_u8(_ptr(packed), n, dim, row_base, _ptr(exc), _ptr(counts),
                                  n_lists, cap, _ptr(out), _stream(stream))
    if st != LBP_OK:
        raise LbpError(st, "lbp_desc_unpack_u8")
    return out
