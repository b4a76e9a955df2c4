"""C-ABI checks that need no GPU: the library loads, exports every symbol that
include/*.h declares, and rejects host-detectable argument errors before
touching the device (SURVEY §8b conventions)."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s+\*?([a-z_][a-z0-9_]*)\s*\(",
                             src, flags=re.M):
            names.append(m.group(1))
    return sorted(set(names))


@pytest.fixture(scope="module")
def L():
    from paper_1504_01883_b200 import build, lbpfused
    build.build()
    return lbpfused.lib()


def test_exports_every_declared_symbol(L):
    names = _declared_functions()
    assert {"lbp_fused_extract", "svm_score", "lbp_descriptor_dim", "lbp_status_string",
            "svm_prepare", "svm_workspace_bytes", "lbp_recognize_host",
            "lbp_recognize_workspace_bytes"} <= set(names)
    for n in names:
        assert hasattr(L, n), n


def test_descriptor_dim_and_status_strings(L):
    from paper_1504_01883_b200 import lbpfused as lb
    assert lb.lbp_descriptor_dim(8, 8, 59) == 3776
    assert lb.lbp_descriptor_dim(1, 1, 256) == 256
    assert L.lbp_descriptor_dim(0, 8, 59) == lb.LBP_E_ARG
    assert L.lbp_descriptor_dim(8, 8, 60) == lb.LBP_E_ARG
    assert L.lbp_descriptor_dim(65536, 65536, 256) == lb.LBP_E_ARG
    for s in range(-6, 1):
        assert lb.status_string(s).startswith("LBP_")


def _geom(lb, n=1, H=8, W=8, pitch=8):
    return lb.lbp_images_t(n, H, W, 0, pitch, pitch, pitch * H, pitch * H)


def test_extract_argument_errors_enqueue_nothing(L):
    """Each host-detectable error returns before any CUDA call (no device is present here)."""
    from paper_1504_01883_b200 import lbpfused as lb
    P = ctypes.c_void_p
    dummy = P(0x1000)  # never dereferenced: validation fails first
    g = _geom(lb)

    def call(grey=dummy, rois=dummy, n=1, dmin=0, dmax=10, cx=2, cy=2, bins=59, desc=dummy, geom=g):
        return L.lbp_fused_extract(grey, None, geom, rois, n, dmin, dmax, cx, cy, bins, desc,
                                   None, None)
    assert call(n=0) == lb.LBP_OK
    assert call(n=-1) == lb.LBP_E_ARG
    assert call(bins=60) == lb.LBP_E_ARG
    assert call(cx=0) == lb.LBP_E_ARG
    assert call(dmin=11) == lb.LBP_E_ARG
    assert call(grey=None) == lb.LBP_E_ARG
    assert call(rois=None) == lb.LBP_E_ARG
    assert call(desc=None) == lb.LBP_E_ARG
    assert call(geom=_geom(lb, pitch=7)) == lb.LBP_E_ARG
    assert call(geom=_geom(lb, n=0)) == lb.LBP_E_ARG
    bad = _geom(lb)
    bad.reserved = 1
    assert call(geom=bad) == lb.LBP_E_ARG


def test_extract_source_argument_errors(L):
    """lbp_extract_source: bad source, missing plane for the source, grey-free depth source
    validated on the depth geometry only."""
    from paper_1504_01883_b200 import lbpfused as lb
    P = ctypes.c_void_p
    dummy = P(0x1000)
    g = _geom(lb)

    def call(source, grey=dummy, depth=dummy, n=1, geom=g):
        return L.lbp_extract_source(grey, depth, geom, dummy, n, 0, 10, 2, 2, 59, source, dummy,
                                    None, None)
    assert call(3) == lb.LBP_E_ARG
    assert call(-1) == lb.LBP_E_ARG
    assert call(lb.LBP_SRC_DEPTH, depth=None) == lb.LBP_E_ARG
    assert call(lb.LBP_SRC_FUSED, depth=None) == lb.LBP_E_ARG
    assert call(lb.LBP_SRC_FUSED, grey=None) == lb.LBP_E_ARG
    assert call(lb.LBP_SRC_GREY, grey=None) == lb.LBP_E_ARG
    assert call(lb.LBP_SRC_DEPTH, n=0) == lb.LBP_OK
    bad = _geom(lb)
    bad.depth_pitch = 7
    assert call(lb.LBP_SRC_DEPTH, grey=None, geom=bad) == lb.LBP_E_ARG


def test_extract_resized_argument_errors(L):
    from paper_1504_01883_b200 import lbpfused as lb
    P = ctypes.c_void_p
    dummy = P(0x1000)
    g = _geom(lb)

    def call(size=64, source=0, grey=dummy, depth=dummy, n=1, geom=g):
        return L.lbp_extract_resized(grey, depth, geom, dummy, n, size, 0, 10, 2, 2, 59, source,
                                     dummy, None, None)
    assert call(size=2) == lb.LBP_E_ARG
    assert call(size=1025) == lb.LBP_E_ARG
    assert call(source=5) == lb.LBP_E_ARG
    assert call(source=lb.LBP_SRC_DEPTH, depth=None) == lb.LBP_E_ARG
    assert call(grey=None) == lb.LBP_E_ARG
    assert call(n=0) == lb.LBP_OK
    big = lb.lbp_images_t(1, 8, (1 << 20) + 1, 0, (1 << 20) + 1, (1 << 20) + 1, 8 << 21, 8 << 21)
    assert call(geom=big) == lb.LBP_E_UNSUPPORTED


def test_svm_train_argument_errors(L):
    from paper_1504_01883_b200 import lbpfused as lb
    P = ctypes.c_void_p
    d = P(0x1000)

    def call(n=4, dim=8, C=2, T=10, inv=100, desc=d):
        return L.svm_train_ovr(desc, n, dim, d, C, d, T, inv, d, d, None, None)
    assert call(T=0) == lb.LBP_E_ARG
    assert call(inv=0) == lb.LBP_E_ARG
    assert call(n=0) == lb.LBP_E_ARG
    assert call(C=0) == lb.LBP_E_ARG
    assert call(desc=None) == lb.LBP_E_ARG
    assert call(T=(1 << 31) + 1) == lb.LBP_E_ARG
    assert call(dim=16385) == lb.LBP_E_UNSUPPORTED


def test_svm_argument_errors(L):
    from paper_1504_01883_b200 import lbpfused as lb
    P = ctypes.c_void_p
    d = P(0x1000)
    call = lambda n=4, dim=8, C=2, desc=d, W=d, b=d, prep=None, pbytes=0: L.svm_score(
        desc, n, dim, W, b, C, prep, pbytes, None, None, None, float("-inf"), None)
    assert call(n=0) == lb.LBP_OK
    # a prepared workspace smaller than svm_workspace_bytes(C, dim) is refused on the host
    need = lb.svm_workspace_bytes(100, 3776)
    assert need > 0
    assert call(dim=3776, C=100, prep=d, pbytes=need - 1) == lb.LBP_E_ARG
    assert call(n=-1) == lb.LBP_E_ARG
    assert call(dim=0) == lb.LBP_E_ARG
    assert call(C=0) == lb.LBP_E_ARG
    assert call(desc=None) == lb.LBP_E_ARG
    assert call(W=None) == lb.LBP_E_ARG
    assert call(b=None) == lb.LBP_E_ARG


def test_recognize_workspace_size(L):
    from paper_1504_01883_b200 import lbpfused as lb
    g = lb.lbp_images_t(16, 128, 128, 0, 128, 128, 128 * 128, 128 * 128)
    n = lb.lbp_recognize_workspace_bytes(g, True, 16, 8, 8, 59)
    assert n >= 16 * 128 * 128 * 3 + 16 * 3776 * 2 + 16 * 20 + 16 * 8
    assert lb.lbp_recognize_workspace_bytes(g, True, 16, 8, 8, 60) == 0


def test_binding_refuses_cpu_tensors():
    import torch
    from paper_1504_01883_b200 import lbpfused as lb
    g = torch.zeros(1, 8, 8, dtype=torch.uint8)
    r = torch.zeros(1, 5, dtype=torch.int32)
    with pytest.raises(ValueError):
        lb.lbp_fused_extract(g, None, r, 0, 10, 2, 2, 59)


def test_desc_pack_host_errors(L):
    from paper_1504_01883_b200 import lbpfused as lb
    fake = ctypes.c_void_p(16)  # never dereferenced: every call below fails validation first
    assert L.lbp_desc_pack_u8(fake, 4, 0, 0, fake, fake, 8, fake, None) == lb.LBP_E_ARG
    assert L.lbp_desc_pack_u8(fake, -1, 8, 0, fake, fake, 8, fake, None) == lb.LBP_E_ARG
    assert L.lbp_desc_pack_u8(fake, 4, 8, 0, fake, fake, -1, fake, None) == lb.LBP_E_ARG
    assert L.lbp_desc_pack_u8(fake, 4, 8, 0, fake, fake, 8, None, None) == lb.LBP_E_ARG
    assert L.lbp_desc_pack_u8(None, 4, 8, 0, fake, fake, 8, fake, None) == lb.LBP_E_ARG
    assert L.lbp_desc_pack_u8(fake, 4, 8, 0, fake, None, 8, fake, None) == lb.LBP_E_ARG
    assert L.lbp_desc_unpack_u8(fake, 4, 0, 0, fake, fake, 1, 8, fake, None) == lb.LBP_E_ARG
    assert L.lbp_desc_unpack_u8(None, 4, 8, 0, fake, fake, 1, 8, fake, None) == lb.LBP_E_ARG
    assert L.lbp_desc_unpack_u8(fake, 4, 8, 0, None, fake, 1, 8, fake, None) == lb.LBP_E_ARG
    assert L.lbp_desc_unpack_u8(fake, 4, 8, 0, fake, fake, -1, 8, fake, None) == lb.LBP_E_ARG
    assert L.lbp_desc_unpack_u8(fake, 0, 8, 0, fake, fake, 1, 8, fake, None) == lb.LBP_OK


def test_extract_gather_argument_errors(L):
    """lbp_extract_gather (the fused database build): destination descriptor checks, all before
    any CUDA call."""
    from paper_1504_01883_b200 import lbpfused as lb
    P = ctypes.c_void_p
    dummy = P(0x1000)
    g = _geom(lb)
    base = 0x10000

    def call(mode=lb.LBP_GATHER_PEERS, bases=(base,), off=0, pitch=64, lab=-1, row0=0, n=1,
             bins=59, scratch=dummy, grey=dummy):
        dst = lb.gather_dst(mode, list(bases), off, pitch, lab, row0)
        return L.lbp_extract_gather(grey, None, g, dummy, n, 0, 10, 1, 1, bins, None, dst,
                                    scratch, None, None)
    assert call(n=0) == lb.LBP_OK
    assert call(mode=0) == lb.LBP_E_ARG
    assert call(mode=lb.LBP_GATHER_MULTIMEM, bases=(base, base)) == lb.LBP_E_ARG
    assert call(bases=(base + 4,)) == lb.LBP_E_ARG
    assert call(bases=(0,)) == lb.LBP_E_ARG
    assert call(off=8) == lb.LBP_E_ARG
    assert call(pitch=56) == lb.LBP_E_ARG   # < dim 59
    assert call(pitch=60) == lb.LBP_E_ARG   # not a multiple of 8
    assert call(lab=2) == lb.LBP_E_ARG
    assert call(row0=-1) == lb.LBP_E_ARG
    assert call(bins=60) == lb.LBP_E_ARG
    assert call(n=-1) == lb.LBP_E_ARG
    assert call(scratch=None) == lb.LBP_E_ARG
    assert call(grey=None) == lb.LBP_E_ARG
    with pytest.raises(ValueError):
        lb.gather_dst(lb.LBP_GATHER_PEERS, [base] * 9, 0, 64, -1, 0)


def test_compact_path_argument_errors(L):
    """lbp_extract_u8 / svm_score_u8 / svm_prepare_u8 (the compact recognition path):
    host-detectable errors return before any CUDA call; exc_cap must cover the bound."""
    from paper_1504_01883_b200 import lbpfused as lb
    P = ctypes.c_void_p
    dummy = P(0x1000)
    g = lb.lbp_images_t(1, 128, 128, 0, 128, 128, 128 * 128, 128 * 128)
    assert lb.lbp_u8_exc_cap_min(g, 3776) == (126 * 126) // 256 == 62
    assert lb.lbp_u8_exc_cap_min(lb.lbp_images_t(1, 2, 2, 0, 2, 2, 4, 4), 59) == 0
    assert lb.lbp_u8_exc_cap_min(_geom(lb, H=400, W=400, pitch=400), 59) == 59  # capped at dim

    def ext(n=1, cap=64, pitch=3776, bins=59, packed=dummy, exc_n=dummy, exc=dummy, grey=dummy):
        return L.lbp_extract_u8(grey, None, g, dummy, n, 0, 10, 8, 8, bins, packed, pitch,
                                exc_n, exc, cap, None, None, None)
    assert ext(n=0) == lb.LBP_OK
    assert ext(cap=61) == lb.LBP_E_ARG        # below the bound
    assert ext(pitch=3775) == lb.LBP_E_ARG    # pitch < dim
    assert ext(bins=60) == lb.LBP_E_ARG
    assert ext(n=-1) == lb.LBP_E_ARG
    assert ext(packed=None) == lb.LBP_E_ARG
    assert ext(exc_n=None) == lb.LBP_E_ARG
    assert ext(exc=None) == lb.LBP_E_ARG
    assert ext(grey=None) == lb.LBP_E_ARG

    def score(n=4, dim=3776, C=10, pitch=3776, cap=64, prep=None, pbytes=0):
        return L.svm_score_u8(dummy, pitch, dummy, dummy, cap, n, dim, dummy, dummy, C, prep,
                              pbytes, None, None, None, 0.0, None)
    assert score(n=0) == lb.LBP_OK
    assert score(n=-1) == lb.LBP_E_ARG
    assert score(C=0) == lb.LBP_E_ARG
    assert score(pitch=100) == lb.LBP_E_ARG
    assert score(dim=70000, pitch=70000) == lb.LBP_E_ARG
    assert score(prep=dummy, pbytes=16) == lb.LBP_E_ARG  # workspace too small
    assert lb.svm_workspace_u8_bytes(100, 3776) > 0
    assert lb.svm_workspace_u8_bytes(100, 40000) == 0    # dim > 32,768: no tensor-core layout
    assert L.svm_prepare_u8(None, 10, 3776, dummy, 1 << 30, None) == lb.LBP_E_ARG
    assert L.svm_prepare_u8(dummy, 10, 3776, dummy, 16, None) == lb.LBP_E_ARG
