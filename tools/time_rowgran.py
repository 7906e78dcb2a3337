import time, torch, sys
sys.path.insert(0, ".")
from paper_2501_02625_b200 import halo as H
b, m, n = 4096, 4096, 4096
for lvl in (1, 2):
    W = (torch.randn(n, m, device="cuda") / 64).bfloat16()
    X = torch.randn(b, m, device="cuda").bfloat16()
    E = (torch.randn(b, n, device="cuda") * 1e-3).bfloat16()
    for gran in (H.GRAN_TENSOR, H.GRAN_ROW):
        layer = H.HaloLinearLayer(W, getattr(H, f"halo{lvl}")(0, 256, gran), out_dtype=torch.bfloat16, grad_dtype=torch.bfloat16)
        ctx = H.SavedContext()
        for _ in range(2):
            layer.forward(X, ctx); layer.backward(ctx, E)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3):
            layer.forward(X, ctx); layer.backward(ctx, E)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 3
        print(f"halo{lvl} gran={gran} b=m=n=4096 fwd+bwd {ms:.3f} ms  ({6*b*m*n/ms/1e9:.1f} TOPS)")
