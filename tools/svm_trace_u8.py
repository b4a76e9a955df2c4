"""Developer tool: phase timestamps of the INT8 compact-descriptor scorer (svm_gemm_u8; build
with LBP_NVCC_EXTRA=-DLBP_SVM_TRACE).  argv: [C=100] [n=16384] [scores=0] [step=0: 1 = each launch follows an extraction of
the batch on the stream, as in bench.py's step].  Prints, for the
first and the last cluster of the last of 3 launches, in us from the earliest stamp: entry,
dependency wait done, first stage ready, last MMA issued, last pass's accumulators complete,
epilogue done, exit."""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
import paper_1504_01883_b200 as lb  # noqa: E402
import synthgen  # noqa: E402

C = int(sys.argv[1]) if len(sys.argv) > 1 else 100
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
want = len(sys.argv) > 3 and sys.argv[3] == "1"
step = len(sys.argv) > 4 and sys.argv[4] == "1"
dev = torch.device('cuda', 0)
g, d = synthgen.gpu_face_crops(n, 128, 128, seed=1, device=dev)
r = torch.from_numpy(synthgen.full_rois(n, 128, 128)).to(dev)
cd = lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59)
W, b = synthgen.svm_weights(C, 3776, seed=1)
W, b = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
ws = lb.svm_prepare_u8(W)
for _ in range(3):
    if step:
        lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59, out=cd)
    lb.svm_score_u8(cd, W, b, prepared=ws, want_scores=want)
torch.cuda.synchronize()
L = lb.lbpfused.lib()
buf = (ctypes.c_ulonglong * 32)()
assert L.lbp_debug_svm_trace(buf) == 0
names = ["entry", "wait_done", "mma_last_issued", "acc_done", "epi_done", "exit", "first_stage"]
t0 = min(v for v in buf if v)
for cl in (0, 1):
    for rk in (0, 1):
        vals = [buf[cl * 16 + rk * 8 + k] for k in range(7)]
        print(("first" if cl == 0 else "last "), "rank", rk,
              " ".join(f"{nm}={(v - t0) / 1e3:.2f}" if v else f"{nm}=-" for nm, v in zip(names, vals)))
