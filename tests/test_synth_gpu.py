"""The GPU input generator draws exactly the crops of the numpy generator."""
import numpy as np
import pytest
import torch

import synthgen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dist", ["face", "constant", "noise"])
@pytest.mark.parametrize("H,W,first", [(128, 128, 0), (64, 64, 1000), (37, 53, 5), (480, 640, 3)])
def test_gpu_generator_bitexact(dist, H, W, first):
    n = 6
    g_ref, d_ref = synthgen.face_crops(n, H, W, seed=42, first_index=first, dist=dist)
    g, d = synthgen.gpu_face_crops(n, H, W, seed=42, first_index=first, dist=dist)
    torch.cuda.synchronize()
    assert np.array_equal(g.cpu().numpy(), g_ref)
    assert np.array_equal(d.cpu().view(torch.int16).numpy().view(np.uint16), d_ref)
