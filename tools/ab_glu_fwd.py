"""Same-process A/B of the SwiGLU GEMM epilogue: the cfg2 MLP step (forward +
backward, 8192 tokens, HALO-2 INT8) with HaloMLP.glu_epi on / off,
interleaved rounds, CUDA-event times, medians.
Usage: python tools/ab_glu_fwd.py [rounds] [steps]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402
from paper_2501_02625_b200.mlp import HaloMLP  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 8
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
b, H, I = 8192, 4096, 14336
g = torch.Generator(device="cuda").manual_seed(0)
bf = torch.bfloat16
wg = (torch.randn(I, H, generator=g, device="cuda") / H ** 0.5).to(bf)
wu = (torch.randn(I, H, generator=g, device="cuda") / H ** 0.5).to(bf)
wd = (torch.randn(H, I, generator=g, device="cuda") / I ** 0.5).to(bf)
x = torch.randn(b, H, generator=g, device="cuda").to(bf)
dy = (torch.randn(b, H, generator=g, device="cuda") * 1e-3).to(bf)
mlp = HaloMLP(wg, wu, wd, halo.halo2(halo.INT8, 256))
res = {True: [], False: []}
fwd = {True: [], False: []}
for r in range(rounds):
    for on in (False, True):
        mlp.glu_epi = on
        for _ in range(3):
            mlp.forward(x)
            mlp.backward(dy)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            mlp.forward(x)
        e1.record()
        for _ in range(steps):
            mlp.forward(x)
            mlp.backward(dy)
        e2.record()
        torch.cuda.synchronize()
        fwd[on].append(e0.elapsed_time(e1) / steps)
        res[on].append(e1.elapsed_time(e2) / steps)
for on in (False, True):
    print(f"glu_epi={int(on)} step_ms median {statistics.median(res[on]):.4f} min {min(res[on]):.4f} "
          f"fwd_ms median {statistics.median(fwd[on]):.4f} min {min(fwd[on]):.4f}")
