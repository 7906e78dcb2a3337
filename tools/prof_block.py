"""Kernel-time breakdown of one cfg3 block step (torch.profiler / CUPTI)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402
from paper_2501_02625_b200.block import LlamaBlock  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "int8"
scheme = None if cfg == "bf16" else (halo.halo2(halo.INT8, 256) if cfg == "int8" else halo.halo2(halo.FP8_E4M3, 256))
blk = LlamaBlock(scheme, bf16=cfg == "bf16")
T = 16384
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randn(T, 4096, generator=g, device="cuda").to(torch.bfloat16)
dy = (torch.randn(T, 4096, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)


def step():
    xi = x.detach().requires_grad_(True)
    y = blk.forward(xi)
    y.backward(dy)
    for l in blk.linears():
        l.grad = None
        l.w.grad = None  # bf16 arm: autograd's dW


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=90))
