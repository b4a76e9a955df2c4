"""Helpers shared by the GPU parity tests (test side only: imports oracle/ and synthgen/)."""
import numpy as np

SVM_RTOL = 1e-5          # J.north_star: "within 1e-5 relative in fp32"
SVM_FLOOR = 2.0 ** -20   # relative floor for near-total cancellation


def svm_tolerance_ok(desc, W, b, s_gpu, s_ref):
    """|s_gpu - s_ref| <= 1e-5 * max(|s_ref|, 2^-20 * (sum_d |x_d w_d| + |b|)) elementwise."""
    mag = np.abs(desc.astype(np.float64)) @ np.abs(W.astype(np.float64)).T + np.abs(b)[None, :]
    scale = np.maximum(np.abs(s_ref.astype(np.float64)), SVM_FLOOR * mag)
    err = np.abs(s_gpu.astype(np.float64) - s_ref.astype(np.float64))
    ok = err <= SVM_RTOL * scale
    return bool(ok.all()), float((err / scale).max()) if err.size else 0.0


def labels_agree_away_from_ties(s_ref, lab_gpu, lab_ref, desc, W, b):
    """Labels must be identical wherever the oracle's top-2 gap exceeds twice the tolerance."""
    if s_ref.shape[1] < 2:
        return bool(np.array_equal(lab_gpu, lab_ref))
    mag = np.abs(desc.astype(np.float64)) @ np.abs(W.astype(np.float64)).T + np.abs(b)[None, :]
    srt = np.sort(s_ref.astype(np.float64), axis=1)
    gap = srt[:, -1] - srt[:, -2]
    tol = SVM_RTOL * np.maximum(np.abs(srt[:, -1]), SVM_FLOOR * mag.max(1))
    clear = gap > 2 * tol
    return bool(np.array_equal(lab_gpu[clear], lab_ref[clear]))
