"""Developer tool: extraction kernel time per variant (config3 shape by default), CUDA events
around K back-to-back launches on one stream (no other kernels in between), inputs larger
than L2.  Prints us per launch and the HBM fraction on the algorithmic bytes (grey + depth
read + the descriptor written) against MEASURED_PEAKS.json.
argv: [crops=16384] [K=50] [variants=u8,u16,fused,depth] [l2: ROIs cycle over 16 images, so
the inputs are L2-resident -- the kernel's compute-only time; hbm: not] [crop size=128]"""
import json
import os
import sys

import torch

sys.path.insert(0, '.')
import paper_1504_01883_b200 as lb  # noqa: E402
import synthgen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
variants = (sys.argv[3] if len(sys.argv) > 3 else "u8,u16,fused,depth").split(",")
dev = torch.device('cuda', 0)
H = int(sys.argv[5]) if len(sys.argv) > 5 else 128
g, d = synthgen.gpu_face_crops(n, H, H, seed=1, device=dev)
if H % 16:  # TMA needs 16-B multiple row pitches: pad the grey rows (200 -> 208 B)
    P = (H + 15) // 16 * 16
    gb = torch.zeros((n, H, P), dtype=torch.uint8, device=dev)
    gb[:, :, :H] = g
    g = gb[:, :, :H]
if H % 8:  # ... and the depth rows (100 px = 200 B -> 208 B)
    P = (H + 7) // 8 * 8
    db = torch.zeros((n, H, P), dtype=torch.uint16, device=dev)
    db[:, :, :H] = d
    d = db[:, :, :H]
r = torch.from_numpy(synthgen.full_rois(n, H, H)).to(dev)
if len(sys.argv) > 4 and sys.argv[4] == "l2":
    r[:, 0] = torch.arange(n, device=dev, dtype=torch.int32) % 16
s = torch.cuda.Stream(dev)
dim = 64 * 59
peak = 6533.2
try:
    peak = json.load(open(os.path.join(os.path.dirname(__file__), '..', 'MEASURED_PEAKS.json')))['hbm_gbs']
except Exception:
    pass
cd = lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59)
out16 = torch.empty((n, dim), dtype=torch.uint16, device=dev)
outf = torch.empty((n, 2 * dim), dtype=torch.uint16, device=dev)
inb = H * H * 3
fns = {
    "u8": (lambda: lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59, out=cd, stream=s), inb + dim + 4),
    "u16": (lambda: lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59, out=out16, stream=s), inb + 2 * dim),
    "fused": (lambda: lb.lbp_extract_source(g, d, r, 600, 1400, 8, 8, 59, lb.LBP_SRC_FUSED, out=outf, stream=s), inb + 4 * dim),
    "depth": (lambda: lb.lbp_extract_source(None, d, r, 600, 1400, 8, 8, 59, lb.LBP_SRC_DEPTH, out=out16, stream=s), H * H * 2 + 2 * dim),
}


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


for v in variants:
    fn, b = fns[v]
    us = timed(fn)
    gbs = n * b / us / 1e3
    print(f"{v}: {us:.1f} us  {gbs:.0f} GB/s  frac {gbs / peak:.3f}  nominal {gbs / 8000:.3f}")
