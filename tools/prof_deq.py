"""One row-granularity HALO-1 backward at b = m = n = 2048 (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2501_02625_b200 import halo as H
b = m = n = 2048
W = (torch.randn(n, m, device="cuda") / 45).bfloat16()
layer = H.HaloLinearLayer(W, H.halo1(0, 256, H.GRAN_ROW), out_dtype=torch.bfloat16, grad_dtype=torch.bfloat16)
ctx = H.SavedContext()
layer.forward(torch.randn(b, m, device="cuda").bfloat16(), ctx)
layer.backward(ctx, (torch.randn(b, n, device="cuda") * 1e-3).bfloat16())
torch.cuda.synchronize()
