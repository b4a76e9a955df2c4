"""Times the tensor-core SVM scorer alone (svm_score with a prepared workspace, labels + top
only, as bench.py calls it) with CUDA events on its stream, for the bench workloads.
Usage: python tools/svm_time.py [n C] ...   (SVM_REAL=1: descriptors of the bench's synthetic
crops instead of random counts 0..8; SVM_CLAMP=1 additionally clamps counts to 255)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1504_01883_b200 as lb
import synthgen

dev = torch.device("cuda", 0)
args = [int(a) for a in sys.argv[1:]] or [16384, 100, 131072, 1000]
D = 3776
for n, C in zip(args[0::2], args[1::2]):
    if os.environ.get("SVM_REAL"):  # real descriptors of the bench's synthetic crops
        gr, dp = synthgen.gpu_face_crops(n, 128, 128, seed=42, device=dev)
        desc = lb.lbp_fused_extract(gr, dp, torch.from_numpy(synthgen.full_rois(n, 128, 128)).to(dev),
                                    600, 1400, 8, 8, 59)
        del gr, dp
        if os.environ.get("SVM_CLAMP"):  # counts above 255 clamped (no high-part corrections)
            desc = desc.view(torch.int16).clamp_(max=255).view(torch.uint16)
    else:
        # counts 0..8: row sums ~15k, like the 126 x 126 interior pixels of a 128 x 128 crop
        g = torch.Generator(device=dev).manual_seed(0)
        desc = torch.randint(0, 9, (n, D), dtype=torch.int16, device=dev, generator=g).view(torch.uint16)
    W, b = synthgen.svm_weights(C, D, seed=1)
    Wt, bt = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
    ws = lb.svm_prepare(Wt)
    lab = torch.empty(n, dtype=torch.int32, device=dev)
    top = torch.empty(n, dtype=torch.float32, device=dev)
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for _ in range(3):
            lb.svm_score(desc, Wt, bt, prepared=ws, want_scores=False, labels=lab, top_score=top,
                         stream=s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record(s)
        for _ in range(reps):
            lb.svm_score(desc, Wt, bt, prepared=ws, want_scores=False, labels=lab, top_score=top,
                         stream=s)
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = 2.0 * n * D * (4 * C + 16 * ((C + 123) // 124))
    # spot check 64 rows against fp64 on the host
    idx = np.linspace(0, n - 1, 64).astype(np.int64)
    x = desc.view(torch.int16)[idx].cpu().numpy().view(np.uint16).astype(np.float64)
    ref = (x @ W.astype(np.float64).T + b.astype(np.float64)).astype(np.float32)
    ok = np.array_equal(ref.max(1), top.cpu().numpy()[idx])
    print(f"n={n} C={C}: svm_score {ms * 1e3:.1f} us  ({flops / ms / 1e9:.0f} TFLOP/s incl. "
          f"ones rows)  top spot-check exact={ok}", flush=True)

