"""Pins for the oracle's SVM on per-block L1-normalised descriptors (SURVEY §8f-3 variant,
S:379-387 normalize).  CPU only."""
import numpy as np
import pytest

import oracle
import synthgen


def test_spec_examples():
    """Single nonzero bin -> that feature is 1.0; a uniform block -> each feature 1/B."""
    B = 59
    h = np.zeros((1, B), np.uint16)
    h[0, 17] = 9
    W = np.zeros((2, B), np.float32)
    W[0, 17] = 0.75
    W[1, :] = 1.0
    b = np.array([0.5, -2.0], np.float32)
    s, lab, top = oracle.svm_score_l1(h, W, b, B)
    assert s[0, 0] == np.float32(1.25) and s[0, 1] == np.float32(-1.0)
    u = np.full((1, B), 3, np.uint16)
    W1 = np.zeros((1, B), np.float32)
    W1[0, 5] = 59.0
    s, _, _ = oracle.svm_score_l1(u, W1, np.zeros(1, np.float32), B)
    assert abs(float(s[0, 0]) - 1.0) <= 1e-6


def test_block_sums_empty_blocks_and_scale_invariance():
    """All-ones W over every block scores (#nonempty blocks) + b; empty blocks contribute 0;
    scaling a block's counts by an integer leaves the features (hence scores) bit-identical."""
    grey, depth = synthgen.face_crops(6, 64, 64, seed=4)
    desc = oracle.lbp_extract(grey, depth, synthgen.full_rois(6, 64, 64), 600, 1400, 8, 8, 59)
    desc[0, :59 * 5] = 0  # five empty cells
    ones = np.ones((1, desc.shape[1]), np.float32)
    s, _, _ = oracle.svm_score_l1(desc, ones, np.array([0.25], np.float32), 59)
    nonempty = (desc.reshape(6, 64, 59).sum(2) > 0).sum(1)
    assert np.allclose(s[:, 0], nonempty + 0.25, rtol=0, atol=1e-5)
    W, b = synthgen.svm_weights(7, desc.shape[1], seed=9)
    s1, l1, _ = oracle.svm_score_l1(desc, W, b, 59)
    scaled = desc.astype(np.int64).reshape(6, 64, 59)
    scaled[:, ::3, :] *= 3  # every third cell x3 (counts stay < 2^16)
    s2, l2, _ = oracle.svm_score_l1(scaled.reshape(6, -1).astype(np.uint16), W, b, 59)
    assert np.array_equal(s1, s2) and np.array_equal(l1, l2)
    zero = np.zeros((1, desc.shape[1]), np.uint16)
    s, _, _ = oracle.svm_score_l1(zero, W, b, 59)
    assert np.array_equal(s[0], b)


def test_equal_block_mass_relates_to_raw_scores():
    """If every block holds N counts, s_l1 = b + (s_raw - b) / N up to fp64 rounding."""
    rng = np.random.default_rng(2)
    n, cells, B, N = 5, 16, 59, 40
    desc = np.zeros((n, cells * B), np.uint16)
    for i in range(n):
        for k in range(cells):
            np.add.at(desc[i], k * B + rng.integers(0, B, N), 1)
    W, b = synthgen.svm_weights(4, cells * B, seed=3)
    s_l1, _, _ = oracle.svm_score_l1(desc, W, b, B)
    s_raw, _, _ = oracle.svm_score(desc, W, b)
    expect = b[None, :].astype(np.float64) + (s_raw.astype(np.float64) - b[None, :]) / N
    assert np.allclose(s_l1, expect, rtol=1e-5, atol=1e-6)


def test_argument_errors():
    h = np.zeros((1, 10), np.uint16)
    W = np.zeros((1, 10), np.float32)
    with pytest.raises(ValueError):
        oracle.svm_score_l1(h, W, np.zeros(1, np.float32), 3)  # 10 % 3 != 0
