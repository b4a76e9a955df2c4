"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times: the whole
batch goes through the same calls as the bench step (persistent TMA extraction kernel, CTA-pair
tensor-core scorer), and sampled crops -- first, last and seeded random indices -- are checked
one by one against the oracle on the SAME crops (the numpy generator reproduces crop i bit for
bit, tests/test_synth_gpu.py): descriptors bit-exact, scores within R13, labels equal away from
ties.  The 2^20-crop case (BASELINE configs[3] total on one GPU) puts descriptor offsets past
2^31 elements."""
import numpy as np
import pytest
import torch

import oracle
import synthgen
from parity_util import labels_agree_away_from_ties, svm_tolerance_ok

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def lb():
    import paper_1504_01883_b200 as lb
    lb.lbpfused.lib()
    return lb


def _full_batch(lb, n, C, n_samples, seed):
    H = W = 128
    grey, depth = synthgen.gpu_face_crops(n, H, W, seed=seed, device=DEV)
    rois = torch.from_numpy(synthgen.full_rois(n, H, W)).to(DEV)
    Wn, bn = synthgen.svm_weights(C, 3776, seed=seed)
    Wt, bt = torch.from_numpy(Wn).to(DEV), torch.from_numpy(bn).to(DEV)
    desc = lb.lbp_fused_extract(grey, depth, rois, 600, 1400, 8, 8, 59)
    scores, labels, top = lb.svm_score(desc, Wt, bt, prepared=lb.svm_prepare(Wt), want_scores=True)
    torch.cuda.synchronize()
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([[0, 1, n // 2, n - 2, n - 1],
                                    rng.integers(0, n, n_samples)])).astype(np.int64)
    it = torch.from_numpy(idx).to(DEV)
    got = desc.index_select(0, it).cpu().view(torch.int16).numpy().view(np.uint16)
    s_got = scores.index_select(0, it).cpu().numpy()
    lab_got = labels.index_select(0, it).cpu().numpy()
    del grey, depth, desc, scores
    torch.cuda.empty_cache()
    # oracle on exactly those crops (crop i is a pure function of (seed, i))
    ref = np.empty_like(got)
    for k, i in enumerate(idx):
        g, d = synthgen.face_crops(1, H, W, seed=seed, first_index=int(i))
        ref[k] = oracle.lbp_extract(g, d, synthgen.full_rois(1, H, W), 600, 1400, 8, 8, 59)[0]
    bad = np.nonzero((got != ref).any(1))[0]
    assert bad.size == 0, f"crops {idx[bad][:5]} differ"
    s_ref, lab_ref, _ = oracle.svm_score(ref, Wn, bn)
    ok, worst = svm_tolerance_ok(ref, Wn, bn, s_got, s_ref)
    assert ok, worst
    assert labels_agree_away_from_ties(s_ref, lab_got, lab_ref, ref, Wn, bn)


def test_config3_full_size(lb):
    """BASELINE configs[2]: 16,384 crops, 100 classes (the bench's default step)."""
    _full_batch(lb, 16384, 100, 48, seed=42)


def test_config4_shard_full_size(lb):
    """BASELINE configs[3] per-GPU shard at 8 GPUs: 131,072 crops, 1,000 classes."""
    _full_batch(lb, 131072, 1000, 24, seed=7)


def test_two_pow_20_crops_int64_offsets(lb):
    """2^20 crops on one GPU (configs[3] total): descriptor element offsets exceed 2^31."""
    free, _ = torch.cuda.mem_get_info()
    if free < 70 * 2**30:
        pytest.skip("needs ~60 GB of free device memory")
    _full_batch(lb, 1 << 20, 10, 16, seed=3)
