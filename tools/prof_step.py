"""Run a few HALO-2 INT8 MLP steps (cfg2 shapes) for ncu captures.
Usage: python tools/prof_step.py [steps] [tokens]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402
from paper_2501_02625_b200.mlp import HaloMLP  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
b = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
H, I = 4096, 14336
g = torch.Generator(device="cuda").manual_seed(0)
bf = torch.bfloat16
wg = (torch.randn(I, H, generator=g, device="cuda") / H ** 0.5).to(bf)
wu = (torch.randn(I, H, generator=g, device="cuda") / H ** 0.5).to(bf)
wd = (torch.randn(H, I, generator=g, device="cuda") / I ** 0.5).to(bf)
x = torch.randn(b, H, generator=g, device="cuda").to(bf)
dy = (torch.randn(b, H, generator=g, device="cuda") * 1e-3).to(bf)
mlp = HaloMLP(wg, wu, wd, halo.halo2(halo.INT8, 256))
for _ in range(steps):
    mlp.forward(x)
    mlp.backward(dy)
torch.cuda.synchronize()
print("done")
