"""H2D bandwidth from pinned host memory: one copy vs the same bytes split over 2 / 4 streams."""
import torch

n = 805_634_048
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for parts in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(parts)]
    step = n // parts
    for rep in range(2):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i, s in enumerate(ss):
            s.wait_event(a)
            with torch.cuda.stream(s):
                d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"parts={parts}: {ms:.2f} ms = {n / ms / 1e6:.1f} GB/s")
