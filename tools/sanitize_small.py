"""Small invocations of every kernel of the library in one process (a fault smoke test; also
the input for compute-sanitizer where it is available -- it is not on this GPU pool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1504_01883_b200 as lb
import synthgen

dev = torch.device("cuda", 0)
g, d = synthgen.gpu_face_crops(150, 128, 128, seed=1, device=dev)
r = torch.from_numpy(synthgen.full_rois(150, 128, 128)).to(dev)
desc = lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59)            # lane59 (TMA)
lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 256)                   # lane256 (256 bins)
lb.lbp_fused_extract(g, None, r, 0, 0, 8, 8, 59)                      # lane59, no depth
lb.lbp_extract_source(g, d, r, 600, 1400, 8, 8, 59, lb.LBP_SRC_FUSED)  # + depth source
lb.lbp_fused_extract(g, d, r[:8].contiguous(), 600, 1400, 8, 8, 59)   # band kernel
gf, df, rf = synthgen.kinect_frames(2, seed=2)
gf, dft = torch.from_numpy(gf).to(dev), torch.from_numpy(df.view(np.int16)).to(dev).view(torch.uint16)
rf = torch.from_numpy(rf).to(dev)
lb.lbp_extract_resized(gf, dft, rf, 200, 600, 1400, 8, 8, 59, lb.LBP_SRC_FUSED)
gb, db, rb = synthgen.kinect_frames(40, seed=4)                           # FRAME variant (160 ROIs)
gb, dbt = torch.from_numpy(gb).to(dev), torch.from_numpy(db.view(np.int16)).to(dev).view(torch.uint16)
lb.lbp_extract_source(gb, dbt, torch.from_numpy(rb).to(dev), 600, 1400, 8, 8, 59, lb.LBP_SRC_FUSED)
for T in (64, 200):                                                       # tile kernels
    gt, dt = synthgen.gpu_face_crops(151, T, T, seed=T, device=dev)
    if T % 16:
        gp = torch.zeros((151, T, 208), dtype=torch.uint8, device=dev)
        gp[:, :, :T] = gt
        gt = gp[:, :, :T]
    rt = torch.from_numpy(synthgen.full_rois(151, T, T)).to(dev)
    rt[::9, 1:] = torch.tensor([3, 2, T - 9, T - 5], dtype=torch.int32)    # generic positions
    lb.lbp_fused_extract(gt, dt, rt, 600, 1400, 8, 8, 59)
cu8 = lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59)                    # compact path
W8, b8 = synthgen.svm_weights(100, 3776, seed=8)
W8t, b8t = torch.from_numpy(W8).to(dev), torch.from_numpy(b8).to(dev)
lb.svm_score_u8(cu8, W8t, b8t, prepared=lb.svm_prepare_u8(W8t))
pk, exc, cnt = lb.desc_pack_u8(desc, row_base=0, cap=64)                  # compaction
lb.desc_unpack_u8(pk, exc, cnt, 64)
for C in (10, 130):
    W, b = synthgen.svm_weights(C, 3776, seed=C)
    Wt, bt = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
    ws = lb.svm_prepare(Wt)
    lb.svm_score(desc, Wt, bt, prepared=ws)                             # tcgen05 fp16 / INT8
    lb.svm_score(desc[:5].contiguous(), Wt, bt)                         # fp64, tiny batch
    lb.svm_score(desc[:40].contiguous(), Wt, bt)                        # fp64, staged
    lb.lbp_recognize(gf, dft, rf, 600, 1400, 8, 8, 59, Wt, bt)          # fused cluster kernel
    lb.svm_score_l1(desc, Wt, bt, 59)
    labels = (torch.arange(150, device=dev) % C).to(torch.int32)
    order = torch.from_numpy(synthgen.train_order(150, 1, seed=3)).to(dev)
    lb.svm_train_ovr(desc, labels, C, order[:60].contiguous(), 100)
torch.cuda.synchronize()
print("sanitize_small: done")
