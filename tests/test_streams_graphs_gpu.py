"""The library's stream contract (include/lbpfused.h: all work enqueued on the caller's stream,
no synchronisation, no mutable global state): calls captured in a CUDA graph replay to the
same results as eager calls, and calls on two concurrent streams give the serial results."""
import numpy as np
import pytest
import torch

import synthgen

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def lb():
    import paper_1504_01883_b200 as lb
    lb.lbpfused.lib()
    return lb


def _batch(n, seed, C):
    grey, depth = synthgen.gpu_face_crops(n, 128, 128, seed=seed, device=DEV)
    rois = torch.from_numpy(synthgen.full_rois(n, 128, 128)).to(DEV)
    W, b = synthgen.svm_weights(C, 3776, seed=seed)
    return grey, depth, rois, torch.from_numpy(W).to(DEV), torch.from_numpy(b).to(DEV)


def test_graph_capture_replays_the_eager_results(lb):
    grey, depth, rois, W, b = _batch(300, 5, 100)
    ws = lb.svm_prepare(W)
    ref_desc = lb.lbp_fused_extract(grey, depth, rois, 600, 1400, 8, 8, 59)
    ref_s, ref_l, ref_t = lb.svm_score(ref_desc, W, b, prepared=ws)
    small = rois[:4].contiguous()
    ref_r = lb.lbp_recognize(grey, depth, small, 600, 1400, 8, 8, 59, W, b)
    torch.cuda.synchronize()
    desc = torch.zeros_like(ref_desc)
    scores = torch.zeros_like(ref_s)
    labels = torch.zeros_like(ref_l)
    top = torch.zeros_like(ref_t)
    r_desc = torch.zeros_like(ref_r[0])
    r_lab = torch.zeros_like(ref_r[2])
    r_top = torch.zeros_like(ref_r[3])
    s = torch.cuda.Stream(DEV)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        lb.lbp_fused_extract(grey, depth, rois, 600, 1400, 8, 8, 59, out=desc, stream=s)
        lb.svm_score(desc, W, b, prepared=ws, scores=scores, labels=labels, top_score=top,
                     stream=s)
        lb.lbp_recognize(grey, depth, small, 600, 1400, 8, 8, 59, W, b, desc=r_desc,
                         labels=r_lab, top_score=r_top, stream=s)
    for _ in range(2):
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(desc.view(torch.int16), ref_desc.view(torch.int16))
        assert torch.equal(scores, ref_s) and torch.equal(labels, ref_l)
        assert torch.equal(top, ref_t)
        assert torch.equal(r_desc.view(torch.int16), ref_r[0].view(torch.int16))
        assert torch.equal(r_lab, ref_r[2]) and torch.equal(r_top, ref_r[3])


def test_two_concurrent_streams_match_serial(lb):
    a = _batch(400, 6, 150)   # INT8 scorer (C > 124)
    bb = _batch(300, 7, 60)   # fp16 scorer
    ws = [lb.svm_prepare(a[3]), lb.svm_prepare(bb[3])]
    ref = []
    for (g, d, r, W, b), w in zip((a, bb), ws):
        desc = lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59)
        ref.append((desc, lb.svm_score(desc, W, b, prepared=w)))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(DEV), torch.cuda.Stream(DEV)]
    outs = []
    for _ in range(3):
        for (g, d, r, W, b), w, s in zip((a, bb), ws, streams):
            desc = lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59, stream=s)
            outs.append((desc, lb.svm_score(desc, W, b, prepared=w, stream=s)))
    torch.cuda.synchronize()
    for k, (desc, (sc, lab, top)) in enumerate(outs):
        rd, (rs, rl, rt) = ref[k % 2]
        assert torch.equal(desc.view(torch.int16), rd.view(torch.int16))
        assert torch.equal(sc, rs) and torch.equal(lab, rl) and torch.equal(top, rt)
