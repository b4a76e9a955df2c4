"""Developer tool: time of the config3 step and of its parts, each as K back-to-back repetitions
between two events (no events between kernels, so the programmatic launches overlap as in
bench.py's step): extraction only, scoring only, extraction + scoring.  argv: [format=u16|u8]
[K=100] [C=100]"""
import sys

import torch

sys.path.insert(0, '.')
import paper_1504_01883_b200 as lb  # noqa: E402
import synthgen  # noqa: E402

fmt = sys.argv[1] if len(sys.argv) > 1 else "u16"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
C = int(sys.argv[3]) if len(sys.argv) > 3 else 100
n = 16384
dev = torch.device('cuda', 0)
g, d = synthgen.gpu_face_crops(n, 128, 128, seed=1, device=dev)
r = torch.from_numpy(synthgen.full_rois(n, 128, 128)).to(dev)
W, b = (torch.from_numpy(a).to(dev) for a in synthgen.svm_weights(C, 3776, seed=1))
lab = torch.empty(n, dtype=torch.int32, device=dev)
top = torch.empty(n, dtype=torch.float32, device=dev)
if fmt == "u8":
    ws = lb.svm_prepare_u8(W)
    bufs = [lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59) for _ in range(2)]
    ext = lambda k: lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59, out=bufs[k & 1])
    sco = lambda k: lb.svm_score_u8(bufs[k & 1], W, b, prepared=ws, want_scores=False,
                                    labels=lab, top_score=top)
else:
    ws = lb.svm_prepare(W)
    bufs = [torch.empty((n, 3776), dtype=torch.uint16, device=dev) for _ in range(2)]
    ext = lambda k: lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59, out=bufs[k & 1])
    sco = lambda k: lb.svm_score(bufs[k & 1], W, b, prepared=ws, want_scores=False,
                                 labels=lab, top_score=top)


def timed(body):
    for k in range(5):
        body(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(K):
        body(k)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1000


te = timed(ext)
ts = timed(sco)
tst = timed(lambda k: (ext(k), sco(k)))
print(f"{fmt}: extraction {te:.1f} us, scoring {ts:.1f} us, sum {te + ts:.1f} us, step {tst:.1f} us")
