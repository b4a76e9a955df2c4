import sys, time, torch
sys.path.insert(0, '.')
import paper_1504_01883_b200 as lb, synthgen
dev = torch.device('cuda', 0)
H = int(sys.argv[3]) if len(sys.argv) > 3 else 200
n = int(sys.argv[1]); reps = int(sys.argv[2])
g, d = synthgen.gpu_face_crops(n, H, H, seed=1, device=dev)
if H % 16:
    gb = torch.zeros((n, H, 208), dtype=torch.uint8, device=dev); gb[:, :, :H] = g; g = gb[:, :, :H]
r = torch.from_numpy(synthgen.full_rois(n, H, H)).to(dev)
out = torch.empty((n, 3776), dtype=torch.uint16, device=dev)
torch.cuda.synchronize()
ref = None
for k in range(reps):
    lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59, out=out)
    torch.cuda.synchronize()
    if ref is None: ref = out.clone()
    elif not torch.equal(out, ref): print('MISMATCH at rep', k, flush=True)
    if k % 50 == 0: print(n, k, 'ok', flush=True)
print('done', flush=True)
