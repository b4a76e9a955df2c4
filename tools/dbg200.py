import sys, time, torch
sys.path.insert(0, '.')
import paper_1504_01883_b200 as lb, synthgen
dev = torch.device('cuda', 0)
H = 200
n = int(sys.argv[1]); seq = sys.argv[2].split(',')
g, d = synthgen.gpu_face_crops(n, H, H, seed=1, device=dev)
gb = torch.zeros((n, H, 208), dtype=torch.uint8, device=dev); gb[:, :, :H] = g; g = gb[:, :, :H]
r = torch.from_numpy(synthgen.full_rois(n, H, H)).to(dev)
torch.cuda.synchronize()
for variant in seq:
    t0 = time.time()
    print(n, variant, 'start', flush=True)
    if variant == 'u16':
        out = lb.lbp_fused_extract(g, d, r, 600, 1400, 8, 8, 59)
    elif variant == 'src':
        out = lb.lbp_extract_source(g, d, r, 600, 1400, 8, 8, 59, lb.LBP_SRC_GREY)
    elif variant == 'u8s':
        sc = torch.empty((n, 3776), dtype=torch.uint16, device=dev)
        out = lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59, scratch=sc)
    else:
        out = lb.lbp_extract_u8(g, d, r, 600, 1400, 8, 8, 59)
    torch.cuda.synchronize()
    print(n, variant, 'ok', time.time() - t0, flush=True)
