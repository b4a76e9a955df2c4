"""Extraction alone on batched 640x480 frames (FRAME variant, ROIs at any column) vs the same
number of 128x128 crops in a stack (aligned boxes), CUDA events, warm."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1504_01883_b200 as lb
import synthgen

dev = torch.device("cuda", 0)


def timeit(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for frames in (240, 1000):
    g, d, r = synthgen.kinect_frames(frames, seed=1)
    g, d = torch.from_numpy(g).to(dev), torch.from_numpy(d.view(np.int16)).to(dev).view(torch.uint16)
    r = torch.from_numpy(r).to(dev)
    n = r.shape[0]
    out = torch.empty((n, 3776), dtype=torch.uint16, device=dev)
    t_frame = timeit(lambda: lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59, out=out))
    gc, dc = synthgen.gpu_face_crops(n, 128, 128, seed=1, device=dev)
    rc = torch.from_numpy(synthgen.full_rois(n, 128, 128)).to(dev)
    t_stack = timeit(lambda: lb.lbp_fused_extract(gc, dc, rc, 600, 1400, 8, 8, 59, out=out))
    print(f"{n} crops: frames (FRAME variant) {t_frame:.1f} us, stack {t_stack:.1f} us")
