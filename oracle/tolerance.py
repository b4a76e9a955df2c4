"""The one definition of "parity" for SVM scores and labels (R13, R14).

TEST INFRASTRUCTURE ONLY (like the rest of ``oracle/``): used by ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s equivalence gate, so all three apply the same
rule.  No arithmetic of the method lives here -- only the comparison of a GPU result with
the oracle's.

R13 (J.north_star "SVM decision values must match within 1e-5 relative in fp32"):
    |s_gpu - s_ref| <= 1e-5 * max(|s_ref|, 2^-20 * (sum_d |x_d w_d| + |b|))
elementwise; the floor only matters under near-total cancellation.
R14 (J.north_star "predicted labels must be identical away from ties"): labels equal
wherever the oracle's top-2 gap exceeds twice the tolerance of the top score.
"""
from __future__ import annotations

import numpy as np

SVM_RTOL = 1e-5          # J.north_star: "within 1e-5 relative in fp32"
SVM_FLOOR = 2.0 ** -20   # relative floor for near-total cancellation


def _magnitude(desc, W, b):
    """sum_d |x_d w_d| + |b_c| per (row, class), in fp64."""
    return (np.abs(np.asarray(desc, np.float64)) @ np.abs(np.asarray(W, np.float64)).T
            + np.abs(np.asarray(b, np.float64))[None, :])


def svm_tolerance_ok(desc, W, b, s_gpu, s_ref):
    """(all within R13, worst err/scale).  desc [n][dim], W [C][dim], b [C], scores [n][C]."""
    mag = _magnitude(desc, W, b)
    scale = np.maximum(np.abs(np.asarray(s_ref, np.float64)), SVM_FLOOR * mag)
    err = np.abs(np.asarray(s_gpu, np.float64) - np.asarray(s_ref, np.float64))
    ok = err <= SVM_RTOL * scale
    return bool(ok.all()), float((err / scale).max()) if err.size else 0.0


def top_score_ok(desc, W, b, top_gpu, s_ref):
    """R13 on the top score alone (the scorer's `top_score` output = max_c s[n][c])."""
    s_ref = np.asarray(s_ref, np.float64)
    if s_ref.shape[0] == 0:
        return True, 0.0
    mag = _magnitude(desc, W, b).max(1)
    top_ref = s_ref.max(1)
    scale = np.maximum(np.abs(top_ref), SVM_FLOOR * mag)
    err = np.abs(np.asarray(top_gpu, np.float64) - top_ref)
    return bool((err <= SVM_RTOL * scale).all()), float((err / scale).max())


def clear_rows(s_ref, desc, W, b):
    """Rows whose oracle top-2 gap exceeds twice the R13 tolerance of the top score."""
    s_ref = np.asarray(s_ref, np.float64)
    if s_ref.shape[1] < 2:
        return np.ones(s_ref.shape[0], bool)
    mag = _magnitude(desc, W, b)
    srt = np.sort(s_ref, axis=1)
    gap = srt[:, -1] - srt[:, -2]
    tol = SVM_RTOL * np.maximum(np.abs(srt[:, -1]), SVM_FLOOR * mag.max(1))
    return gap > 2 * tol


def labels_agree_away_from_ties(s_ref, lab_gpu, lab_ref, desc, W, b):
    """Labels must be identical wherever the oracle's top-2 gap exceeds twice the tolerance."""
    clear = clear_rows(s_ref, desc, W, b)
    return bool(np.array_equal(np.asarray(lab_gpu)[clear], np.asarray(lab_ref)[clear]))


def check_svm(desc, W, b, s_ref, lab_ref, lab_gpu, s_gpu=None, top_gpu=None):
    """The whole R13 + R14 check used by smoke() and bench's gate.  Returns (ok, detail)."""
    detail = {}
    ok = True
    if s_gpu is not None:
        good, worst = svm_tolerance_ok(desc, W, b, s_gpu, s_ref)
        detail["scores_worst_rel"] = worst
        ok &= good
    if top_gpu is not None:
        good, worst = top_score_ok(desc, W, b, top_gpu, s_ref)
        detail["top_worst_rel"] = worst
        ok &= good
    lab_ok = labels_agree_away_from_ties(s_ref, lab_gpu, lab_ref, desc, W, b)
    detail["labels_ok"] = lab_ok
    detail["rows_clear"] = int(clear_rows(s_ref, desc, W, b).sum())
    return bool(ok and lab_ok), detail
