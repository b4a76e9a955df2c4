"""B200-native fused-depth LBP descriptor + linear-SVM hot path of arXiv 1504.01883.

The computation lives in the sm_100a CUDA library ``liblbpfused.so`` behind the
C ABI of ``include/lbpfused.h``; ``lbpfused`` is its thin ctypes binding.
"""
from .lbpfused import (LBP_E_ARG, LBP_E_CUDA, LBP_E_GRID, LBP_E_OVERFLOW, LBP_E_ROI,
                       LBP_E_UNSUPPORTED, LBP_OK, LBP_SRC_DEPTH, LBP_SRC_FUSED, LBP_SRC_GREY,
                       CompactDesc, LbpError, desc_pack_u8, desc_unpack_u8, gather_dst, images_geometry, lbp_descriptor_dim, lbp_extract_resized,
                       lbp_extract_gather, lbp_extract_source, lbp_extract_u8, lbp_u8_exc_cap_min,
                       lbp_fused_extract, lbp_recognize, lbp_recognize_host,
                       lbp_recognize_workspace_bytes,
                       status_string, svm_prepare, svm_score, svm_score_l1,
                       svm_prepare_u8, svm_score_u8, svm_train_ovr, svm_workspace_bytes,
                       svm_workspace_u8_bytes)

__all__ = ["LBP_OK", "LBP_E_ARG", "LBP_E_ROI", "LBP_E_GRID", "LBP_E_OVERFLOW",
           "LBP_SRC_GREY", "LBP_SRC_DEPTH", "LBP_SRC_FUSED", "lbp_extract_source",
           "lbp_extract_resized", "lbp_recognize",
           "LBP_E_UNSUPPORTED", "LBP_E_CUDA", "LbpError", "images_geometry",
           "desc_pack_u8", "desc_unpack_u8", "gather_dst", "lbp_extract_gather",
           "lbp_descriptor_dim", "lbp_fused_extract", "lbp_recognize_host",
           "lbp_recognize_workspace_bytes", "status_string", "svm_prepare", "svm_score",
           "svm_score_l1", "svm_train_ovr", "svm_workspace_bytes", "CompactDesc",
           "lbp_extract_u8", "lbp_u8_exc_cap_min", "svm_prepare_u8", "svm_score_u8",
           "svm_workspace_u8_bytes"]
