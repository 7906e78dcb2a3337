"""Driver for the ncu capture of the large-block kernels: K1 at B = 512 (the
one-exchange path in the v4 kernel) and K2 at B = 1024 (fwht_cols_lb.cu),
8192 x 8192 bf16, phase A + phase B each, after one warm-up call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402

x = torch.randn(8192, 8192, device="cuda").to(torch.bfloat16)
e = (torch.randn(8192, 8192, device="cuda") * 1e-3).to(torch.bfloat16)
for _ in range(2):
    halo.rotate_quantize(x, 512)
    halo.left_rotate_quantize(e, 1024)
torch.cuda.synchronize()
print("ok")
