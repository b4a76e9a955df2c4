"""GPU parity of svm_train_ovr against the oracle: the integer state z and the
fp32 model are BIT-EXACT (the training is defined in exact integers, R20) for
59- and 256-bin descriptors, more classes than CTAs, labels outside [0, C); the trained model
scores its separable training set correctly with svm_score."""
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


def _dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV).to(dtype)


def _check(lb, desc, labels, C, order, inv_lambda):
    W, b, z = lb.svm_train_ovr(
        torch.from_numpy(desc.view(np.int16)).to(DEV).view(torch.uint16),
        _dev(labels, torch.int32), C, _dev(order, torch.int32), inv_lambda, return_z=True)
    torch.cuda.synchronize()
    Wr, br, zr = oracle.svm_train_ovr(desc, labels, C, order, inv_lambda, return_z=True)
    assert np.array_equal(z.cpu().numpy(), zr)
    assert np.array_equal(W.cpu().numpy().view(np.uint32), Wr.view(np.uint32))
    assert np.array_equal(b.cpu().numpy().view(np.uint32), br.view(np.uint32))
    return W, b


@pytest.mark.parametrize("bins,n,C,epochs,inv_lambda", [(59, 60, 5, 3, 1000), (59, 33, 1, 2, 7),
                                                        (256, 12, 3, 2, 10000)])
def test_descriptors(lb, bins, n, C, epochs, inv_lambda):
    grey, depth = synthgen.face_crops(n, 64, 64, seed=n)
    desc = oracle.lbp_extract(grey, depth, synthgen.full_rois(n, 64, 64), 600, 1400, 8, 8, bins)
    labels = (np.arange(n) % (C + 1)).astype(np.int32)  # label C: a negative for every class
    _check(lb, desc, labels, C, synthgen.train_order(n, epochs, seed=n), inv_lambda)


def test_more_classes_than_ctas(lb):
    rng = np.random.default_rng(3)
    n, dim, C = 40, 236, 350
    desc = rng.integers(0, 12, (n, dim)).astype(np.uint16)
    labels = rng.integers(0, C, n).astype(np.int32)
    _check(lb, desc, labels, C, synthgen.train_order(n, 2, seed=3), 50)


def test_trained_model_recognises_separable_clusters(lb):
    rng = np.random.default_rng(4)
    C, per, dim = 6, 10, 59 * 8
    X, labels = [], []
    for c in range(C):
        base = rng.integers(0, 3, (per, dim))
        base[:, c * 59:(c + 1) * 59] += 15
        X.append(base)
        labels += [c] * per
    X = np.concatenate(X).astype(np.uint16)
    labels = np.array(labels, np.int32)
    W, b = _check(lb, X, labels, C, synthgen.train_order(len(X), 20, seed=4), 100)
    _, pred, _ = lb.svm_score(torch.from_numpy(X.view(np.int16)).to(DEV).view(torch.uint16), W, b)
    assert np.array_equal(pred.cpu().numpy(), labels)


@pytest.mark.parametrize("dim,n,epochs", [(59, 30, 3),        # odd dim: smem-z kernel
                                          (120, 40, 820),     # T = 32,800: int64 register z
                                          (16384, 6, 2)])     # 1,024-thread register kernel
def test_kernel_variants(lb, dim, n, epochs):
    rng = np.random.default_rng(dim + n)
    desc = rng.integers(0, 300, (n, dim)).astype(np.uint16)
    labels = rng.integers(0, 4, n).astype(np.int32)
    _check(lb, desc, labels, 3, synthgen.train_order(n, epochs, seed=dim), 97)
