"""Does a CUDA graph captured with torch record the library's launches (cudart static)?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1504_01883_b200 as lb
import synthgen

dev = torch.device("cuda", 0)
g, d = synthgen.face_crops(4, 128, 128, seed=1)
grey = torch.from_numpy(g).to(dev)
depth = torch.from_numpy(d.view(np.int16)).to(dev).view(torch.uint16)
rois = torch.from_numpy(synthgen.full_rois(4, 128, 128)).to(dev)
out = torch.zeros((4, 3776), dtype=torch.uint16, device=dev)
s = torch.cuda.Stream(dev)
ref = lb.lbp_fused_extract(grey, depth, rois, 600, 1400, 8, 8, 59)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=s):
    lb.lbp_fused_extract(grey, depth, rois, 600, 1400, 8, 8, 59, out=out, stream=s)
torch.cuda.synchronize()
print("after capture, out nonzero:", int(out.view(torch.int16).ne(0).sum()))
graph.replay()
torch.cuda.synchronize()
print("after replay, equal to eager:", bool(torch.equal(out.view(torch.int16), ref.view(torch.int16))))
