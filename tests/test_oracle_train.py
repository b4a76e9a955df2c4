"""Pins for the oracle's one-vs-rest linear SVM training (
DESIGN.md reading R20: Pegasos steps 1/(lambda t) over a seeded visit order, bias folded in as
a constant feature, computed exactly in integers).  CPU only."""
from fractions import Fraction as F

import numpy as np
import pytest

import oracle
import synthgen


def _pegasos_rational(X, y, order, inv_lambda):
    """Textbook Pegasos in exact rationals: w_t = (1 - 1/t) w_{t-1} + [viol] y x~ / (lambda t),
    viol iff t == 1 or y (w_{t-1} . x~) < 1, x~ = (x, 1), lambda = 1 / inv_lambda."""
    lam = F(1, inv_lambda)
    dim = X.shape[1]
    w = [F(0)] * (dim + 1)
    for t, i in enumerate(order, start=1):
        xt = [int(v) for v in X[i]] + [1]
        viol = t == 1 or y[i] * sum(a * b for a, b in zip(w, xt)) < 1
        w = [(1 - F(1, t)) * a for a in w]
        if viol:
            w = [a + F(y[i]) * b / (lam * t) for a, b in zip(w, xt)]
    return w


@pytest.mark.parametrize("seed,inv_lambda,epochs", [(1, 10, 3), (2, 1000, 4), (3, 1, 2)])
def test_integer_form_equals_rational_pegasos(seed, inv_lambda, epochs):
    rng = np.random.default_rng(seed)
    n, dim, C = 17, 6, 3
    X = rng.integers(0, 9, (n, dim)).astype(np.uint16)
    labels = rng.integers(0, C, n).astype(np.int32)
    order = synthgen.train_order(n, epochs, seed=seed)
    W, b, z = oracle.svm_train_ovr(X, labels, C, order, inv_lambda, return_z=True)
    for c in range(C):
        y = np.where(labels == c, 1, -1)
        w = _pegasos_rational(X, y, order, inv_lambda)
        T = order.size
        assert [int(v) for v in z[c]] == [a * T / inv_lambda for a in w]  # z = lambda T w
        assert np.array_equal(W[c], np.array([float(a) for a in w[:dim]], np.float32))
        assert b[c] == np.float32(float(w[dim]))


def test_two_point_problem_separates():
    """S:456 example (u16 features): positives {(2,0)}, negatives {(0,2)}."""
    X = np.array([[2, 0], [0, 2]], np.uint16)
    labels = np.array([0, 1], np.int32)
    W, b = oracle.svm_train_ovr(X, labels, 2, synthgen.train_order(2, 50, seed=1), 10)
    s = X.astype(np.float64) @ W.T.astype(np.float64) + b
    assert s[0, 0] > 0 > s[1, 0] and s[1, 1] > 0 > s[0, 1]


def test_separable_clusters_zero_training_error_and_objective():
    """well-separated clusters -> every training sample predicted as its own label;
    S:487: final objective <= objective at w = 0, b = 0 (= 1)."""
    rng = np.random.default_rng(4)
    C, per, dim = 4, 12, 40
    X, labels = [], []
    for c in range(C):
        base = rng.integers(0, 3, (per, dim))
        base[:, c * 10:(c + 1) * 10] += 20  # the class's own block of bins
        X.append(base)
        labels += [c] * per
    X = np.concatenate(X).astype(np.uint16)
    labels = np.array(labels, np.int32)
    inv_lambda = 100
    W, b = oracle.svm_train_ovr(X, labels, C, synthgen.train_order(len(X), 30, seed=4),
                                inv_lambda)
    _, pred, _ = oracle.svm_score(X, W, b)
    assert np.array_equal(pred, labels)
    for c in range(C):
        y = np.where(labels == c, 1.0, -1.0)
        margin = y * (X.astype(np.float64) @ W[c].astype(np.float64) + b[c])
        obj = 0.5 / inv_lambda * (np.sum(W[c].astype(np.float64) ** 2) + float(b[c]) ** 2) + \
            np.maximum(0.0, 1.0 - margin).mean()
        assert obj <= 1.0


def test_determinism_order_and_errors():
    rng = np.random.default_rng(5)
    X = rng.integers(0, 5, (30, 8)).astype(np.uint16)
    labels = rng.integers(0, 3, 30).astype(np.int32)
    o1 = synthgen.train_order(30, 5, seed=7)
    a = oracle.svm_train_ovr(X, labels, 3, o1, 50)
    b = oracle.svm_train_ovr(X, labels, 3, o1, 50)
    assert all(np.array_equal(p, q) for p, q in zip(a, b))
    assert np.array_equal(np.sort(o1[:30]), np.arange(30))  # each epoch is a permutation
    with pytest.raises(ValueError):
        oracle.svm_train_ovr(X, labels, 3, np.array([0, 30], np.int32), 50)
    with pytest.raises(ValueError):
        oracle.svm_train_ovr(X, labels, 3, o1, 0)
