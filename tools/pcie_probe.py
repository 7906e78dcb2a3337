"""H2D / D2H pinned-copy bandwidth on the box (context for bench.py's e2e)."""
import torch
n = 134217728
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n // 2, dtype=torch.uint8, pin_memory=True)
d2 = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
def t(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record(); fn(); b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)
ms = t(lambda: d.copy_(h, non_blocking=True)); print("H2D 134MB", round(ms, 3), "ms", round(n / ms / 1e6, 1), "GB/s")
ms = t(lambda: h2.copy_(d2, non_blocking=True)); print("D2H 67MB", round(ms, 3), "ms", round(n / 2 / ms / 1e6, 1), "GB/s")
def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
ms = t(both); print("H2D 134MB || D2H 67MB", round(ms, 3), "ms")
