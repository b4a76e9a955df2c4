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


def _crop_batch(n, T, seed):
    grey, depth = synthgen.gpu_face_crops(n, T, T, seed=seed, device=DEV)
    return grey, depth, torch.from_numpy(synthgen.full_rois(n, T, T)).to(DEV)


@pytest.mark.parametrize("form,T,C", [("u16", 128, 100), ("u8", 128, 100), ("u8", 128, 1000),
                                      ("u16", 64, 100)])
def test_back_to_back_steps_share_one_descriptor_buffer(lb, form, T, C):
    """The extraction kernels are launched as programmatic dependents of the previous kernel on
    the stream and the scorers let them be scheduled early (ptx.cuh: launch_dependents /
    grid_dependency_wait): step k+1's extraction may start while step k's scorer still reads
    the descriptor buffer it overwrites.  Twenty back-to-back extract -> score steps over two
    alternating batches through ONE descriptor buffer, no synchronisation in between, must
    reproduce the labels and top scores of isolated, synchronised runs."""
    n = 4096
    batches = [_crop_batch(n, T, seed) for seed in (11, 12)]
    W, b = (torch.from_numpy(a).to(DEV) for a in synthgen.svm_weights(C, 3776, seed=C))
    if form == "u16":
        ws = lb.svm_prepare(W)
        buf = torch.empty((n, 3776), dtype=torch.uint16, device=DEV)

        def step(g, d, r, labels, top):
            lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59, out=buf)
            lb.svm_score(buf, W, b, prepared=ws, want_scores=False, labels=labels,
                         top_score=top)
    else:
        ws = lb.svm_prepare_u8(W)
        buf = lb.lbp_extract_u8(*batches[0], 600, 1400, 8, 8, 59)  # (allocates)

        def step(g, d, r, labels, top):
            lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59, out=buf)
            lb.svm_score_u8(buf, W, b, prepared=ws, want_scores=False, labels=labels,
                            top_score=top)
    ref = []
    for g, d, r in batches:
        lab = torch.empty(n, dtype=torch.int32, device=DEV)
        top = torch.empty(n, dtype=torch.float32, device=DEV)
        step(g, d, r, lab, top)
        torch.cuda.synchronize()
        ref.append((lab, top))
    assert not torch.equal(ref[0][0], ref[1][0])  # the two batches are told apart
    outs = [(torch.empty(n, dtype=torch.int32, device=DEV),
             torch.empty(n, dtype=torch.float32, device=DEV)) for _ in range(20)]
    for k, (lab, top) in enumerate(outs):
        step(*batches[k & 1], lab, top)
    torch.cuda.synchronize()
    for k, (lab, top) in enumerate(outs):
        assert torch.equal(lab, ref[k & 1][0]), f"step {k}: labels"
        assert torch.equal(top, ref[k & 1][1]), f"step {k}: top scores"


def test_extraction_reads_what_the_previous_extraction_wrote(lb):
    """Read-after-write across two programmatic-dependent launches: the second extraction's
    grey images ARE the first extraction's descriptor buffer (16,384 rows of 7,552 B viewed as
    7,552 crops of 128 x 128 B).  The first kernel lets its dependent be scheduled at once, so
    the second one's CTAs start as the first one's exit; their loads must still see every row
    (compared with the same launches separated by a synchronisation)."""
    n1 = 16384
    g1, d1, r1 = _crop_batch(n1, 128, 21)
    buf = torch.empty((n1, 3776), dtype=torch.uint16, device=DEV)
    n2 = n1 * 7552 // (128 * 128)
    grey2 = buf.view(torch.uint8).view(n2, 128, 128)
    r2 = torch.from_numpy(synthgen.full_rois(n2, 128, 128)).to(DEV)
    out = torch.empty((n2, 3776), dtype=torch.uint16, device=DEV)
    lb.lbp_fused_extract(g1, d1, r1, 600, 1400, 8, 8, 59, out=buf)
    torch.cuda.synchronize()
    ref = lb.lbp_fused_extract(grey2, None, r2, 0, 0, 8, 8, 59)
    torch.cuda.synchronize()
    for _ in range(5):
        buf.zero_()
        lb.lbp_fused_extract(g1, d1, r1, 600, 1400, 8, 8, 59, out=buf)
        lb.lbp_fused_extract(grey2, None, r2, 0, 0, 8, 8, 59, out=out)
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), ref.view(torch.int16))
