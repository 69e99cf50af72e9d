"""H2D bandwidth from pinned memory: one stream vs two (x and y arrays on
separate copy streams), 160 MB each, as the e2e leg moves them."""
import torch
n = 20_000_000
hx = torch.empty(n, dtype=torch.float64).pin_memory()
hy = torch.empty(n, dtype=torch.float64).pin_memory()
dx = torch.empty(n, dtype=torch.float64, device="cuda")
dy = torch.empty_like(dx)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("one stream", "two streams", "one stream", "two streams"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if mode == "one stream":
        dx.copy_(hx, non_blocking=True)
        dy.copy_(hy, non_blocking=True)
    else:
        s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s1):
            dx.copy_(hx, non_blocking=True)
        with torch.cuda.stream(s2):
            dy.copy_(hy, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{mode}: {ms:.3f} ms  {320e6 / ms / 1e6:.1f} GB/s")
