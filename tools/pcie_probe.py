"""PCIe probe: pinned H2D / D2H bandwidth alone and concurrently (the e2e floor)."""
import torch
n = 157286400
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
o = torch.empty(77500416, dtype=torch.uint8, device="cuda")
ho = torch.empty(77500416, dtype=torch.uint8).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best
h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: ho.copy_(o, non_blocking=True))
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(o, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
bo = t(both)
print(f"H2D {n/h2d/1e6:.1f} GB/s ({h2d:.3f} ms)  D2H {ho.numel()/d2h/1e6:.1f} GB/s ({d2h:.3f} ms)  both {bo:.3f} ms")
