"""Host-side cost of one cfg2 MLP step: time to ENQUEUE a step on the CPU
(no synchronisation) against its device time.  If enqueue >= device, the
step is launch-bound and the e2e loop's extra host work shows up in e2e.
  python tools/host_overhead.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402
from paper_2501_02625_b200.mlp import HaloMLP  # noqa: E402

H, I, T = 4096, 14336, 8192
g = torch.Generator(device="cuda").manual_seed(0)
bf = torch.bfloat16
wg = (torch.randn(I, H, generator=g, device="cuda") / H ** 0.5).to(bf)
wu = (torch.randn(I, H, generator=g, device="cuda") / H ** 0.5).to(bf)
wd = (torch.randn(H, I, generator=g, device="cuda") / I ** 0.5).to(bf)
x = torch.randn(T, H, generator=g, device="cuda").to(bf)
dy = (torch.randn(T, H, generator=g, device="cuda") * 1e-3).to(bf)
mlp = HaloMLP(wg, wu, wd, halo.halo2(halo.INT8, 256))
for _ in range(5):
    mlp.forward(x)
    mlp.backward(dy)
torch.cuda.synchronize()
# block the GPU so the CPU enqueue is measured without back-pressure
n = 10
torch.cuda._sleep(int(2e9))  # ~1 s of device spin
t0 = time.perf_counter()
for _ in range(n):
    mlp.forward(x)
    mlp.backward(dy)
t1 = time.perf_counter()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(n):
    mlp.forward(x)
    mlp.backward(dy)
b.record()
torch.cuda.synchronize()
print(f"host enqueue {1e3 * (t1 - t0) / n:.3f} ms/step, device {a.elapsed_time(b) / n:.3f} ms/step")
