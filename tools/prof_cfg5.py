"""torch.profiler breakdown of one cfg5 step (HqFsdpLlama), top kernels by
device time.  python tools/prof_cfg5.py [layers]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402
from paper_2501_02625_b200.train import HqFsdpLlama, LlamaDims  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
d = LlamaDims(layers=L)
m = HqFsdpLlama(d, halo.halo2(halo.INT8, 256))
x = torch.randn(8192, d.hidden, device="cuda").to(torch.bfloat16)
dy = (torch.randn(8192, d.hidden, device="cuda") * 1e-3).to(torch.bfloat16)
for _ in range(2):
    m.step(x, dy)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    m.step(x, dy)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=40, max_name_column_width=90))
