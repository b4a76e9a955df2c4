"""GPU parity of svm_score_l1 (SVM on per-block L1-normalised descriptors, SURVEY §8f-3
variant) against the oracle: scores within the R13-style tolerance on the normalised
features, labels equal away from ties; 59-bin (8 crops per CTA) and 256-bin (1 crop per CTA)
descriptors, empty blocks and rows, C from 1 to 200."""
import numpy as np
import pytest
import torch

import oracle
import synthgen

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def lb():
    import paper_1504_01883_b200 as lb
    lb.lbpfused.lib()
    return lb


def _features(desc, block):
    h = desc.astype(np.float64).reshape(desc.shape[0], -1, block)
    N = h.sum(2, keepdims=True)
    return np.where(N > 0, h / np.where(N > 0, N, 1), 0.0).reshape(desc.shape[0], -1)


@pytest.mark.parametrize("bins,C", [(59, 1), (59, 10), (59, 200), (256, 7)])
def test_l1_scores(lb, bins, C):
    grey, depth = synthgen.face_crops(21, 64, 64, seed=bins + C)
    desc = oracle.lbp_extract(grey, depth, synthgen.full_rois(21, 64, 64), 600, 1400, 8, 8, bins)
    desc[3, : bins * 10] = 0   # empty blocks
    desc[7] = 0                # empty row -> bias
    W, b = synthgen.svm_weights(C, desc.shape[1], seed=C)
    s_ref, lab_ref, top_ref = oracle.svm_score_l1(desc, W, b, bins)
    s, lab, top = lb.svm_score_l1(
        torch.from_numpy(desc.view(np.int16)).to(DEV).view(torch.uint16),
        torch.from_numpy(W).to(DEV), torch.from_numpy(b).to(DEV), bins)
    s, lab = s.cpu().numpy(), lab.cpu().numpy()
    f = _features(desc, bins)
    mag = np.abs(f) @ np.abs(W.astype(np.float64)).T + np.abs(b)[None, :]
    tol = 1e-5 * np.maximum(np.abs(s_ref.astype(np.float64)), 2.0 ** -20 * mag)
    assert (np.abs(s.astype(np.float64) - s_ref) <= tol).all()
    if C > 1:
        srt = np.sort(s_ref, axis=1)
        clear = (srt[:, -1] - srt[:, -2]) > 2 * tol.max(1)
        assert np.array_equal(lab[clear], lab_ref[clear])
    assert np.array_equal(s[7], b)
