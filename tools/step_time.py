"""Developer tool: where the recognition step's time goes (config3 shape by default).
Times, with CUDA events around K back-to-back launches (no events in between):
  ext    lbp_extract_u8 alone            svm   svm_score_u8 alone (labels + top)
  step   eager extract + score           graph the same step captured in a CUDA graph
  host   the Python binding's CPU time per eager step (no GPU sync)
argv: [classes=100] [crops=16384] [K=50]"""
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_1504_01883_b200 as lb  # noqa: E402
import synthgen  # noqa: E402

C = int(sys.argv[1]) if len(sys.argv) > 1 else 100
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
K = int(sys.argv[3]) if len(sys.argv) > 3 else 50
dev = torch.device('cuda', 0)
g, d = synthgen.gpu_face_crops(n, 128, 128, seed=1, device=dev)
r = torch.from_numpy(synthgen.full_rois(n, 128, 128)).to(dev)
cd = lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59)
W, b = synthgen.svm_weights(C, 3776, seed=1)
W, b = torch.from_numpy(W).to(dev), torch.from_numpy(b).to(dev)
ws = lb.svm_prepare_u8(W)
lab = torch.empty(n, dtype=torch.int32, device=dev)
top = torch.empty(n, dtype=torch.float32, device=dev)
s = torch.cuda.Stream(dev)


def ext():
    lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59, out=cd, stream=s)


def svm():
    lb.svm_score_u8(cd, W, b, prepared=ws, want_scores=False, labels=lab, top_score=top, stream=s)


def step():
    ext()
    svm()


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(K):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3


res = {"ext": timed(ext), "svm": timed(svm), "step": timed(step)}
graph = torch.cuda.CUDAGraph()
torch.cuda.synchronize()
with torch.cuda.graph(graph, stream=s):
    step()
torch.cuda.synchronize()
def replay():
    with torch.cuda.stream(s):
        graph.replay()


res["graph"] = timed(replay)
graph10 = torch.cuda.CUDAGraph()
torch.cuda.synchronize()
with torch.cuda.graph(graph10, stream=s):
    for _ in range(10):
        step()
torch.cuda.synchronize()


def replay10():
    with torch.cuda.stream(s):
        graph10.replay()


res["graph10_per_step"] = timed(replay10) / 10
t0 = time.perf_counter()
for _ in range(K):
    step()
res["host"] = (time.perf_counter() - t0) / K * 1e6
torch.cuda.synchronize()
print(" ".join(f"{k}={v:.1f}us" for k, v in res.items()))
