"""Developer tool: phase timestamps of the fp16 SVM kernel (build with
LBP_NVCC_EXTRA=-DLBP_SVM_TRACE; prints entry / prologue / MMA / epilogue / exit times in us
of the first and the last cluster of the last of 3 launches at config3 size).  argv: [step=0:
1 = each launch follows an extraction of the batch on the stream, as in bench.py's step]."""
import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_1504_01883_b200 as lb, synthgen
dev = torch.device('cuda', 0)
g, d = synthgen.gpu_face_crops(16384, 128, 128, seed=1, device=dev)
r = torch.from_numpy(synthgen.full_rois(16384, 128, 128)).to(dev)
desc = lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59)
W, b = synthgen.svm_weights(100, 3776, seed=1)
W, b = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
ws = lb.svm_prepare(W)
step = len(sys.argv) > 1 and sys.argv[1] == "1"
for i in range(3):
    if step:
        lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59, out=desc)
    lb.svm_score(desc, W, b, prepared=ws, want_scores=False)
torch.cuda.synchronize()
import ctypes
L = lb.lbpfused.lib()
buf = (ctypes.c_ulonglong * 32)()
assert L.lbp_debug_svm_trace(buf) == 0
names = ["entry", "prologue_done", "mma_issued", "mma_done", "epilogue_done", "exit"]
t0 = min(v for v in buf if v)
for cl in (0, 1):
    for rk in (0, 1):
        vals = [buf[cl * 16 + rk * 8 + k] for k in range(6)]
        print(("first" if cl == 0 else "last "), "rank", rk,
              " ".join(f"{n}={(v - t0) / 1e3:.2f}" if v else f"{n}=-" for n, v in zip(names, vals)))
