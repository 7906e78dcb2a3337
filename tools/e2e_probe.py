"""Where bench.py's e2e loses to the device-only step (cfg2 MLP, 20 steps):
(a) device-only steps, (b) the same steps with the per-step H2D (X, dY) and
D2H (dX) byte volume copied on side streams but NO dependencies (pure PCIe /
copy-engine interference), (c) bench.py's double-buffered e2e loop."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402
from paper_2501_02625_b200.mlp import HaloMLP  # noqa: E402

b, H, I, K = 8192, 4096, 14336, 20
g = torch.Generator(device="cuda").manual_seed(0)
bf = torch.bfloat16
wg = (torch.randn(I, H, generator=g, device="cuda") / H ** 0.5).to(bf)
wu = (torch.randn(I, H, generator=g, device="cuda") / H ** 0.5).to(bf)
wd = (torch.randn(H, I, generator=g, device="cuda") / I ** 0.5).to(bf)
x = torch.randn(b, H, generator=g, device="cuda").to(bf)
dy = (torch.randn(b, H, generator=g, device="cuda") * 1e-3).to(bf)
mlp = HaloMLP(wg, wu, wd, halo.halo2(halo.INT8, 256))
hx, hdy = x.cpu().pin_memory(), dy.cpu().pin_memory()
hdx = torch.empty((b, H), dtype=bf, pin_memory=True)
xs, dys = torch.empty_like(x), torch.empty_like(dy)
cs, ds = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()


def timed(fn):
    for _ in range(3):
        fn(2)
    torch.cuda.synchronize()
    out = []
    for _ in range(3):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn(K)
        e.record()
        torch.cuda.synchronize()
        out.append(round(a.elapsed_time(e) / K, 4))
    return out


def dev(n):
    for _ in range(n):
        mlp.forward(x)
        mlp.backward(dy)


def interfere(n):
    for _ in range(n):
        with torch.cuda.stream(cs):
            xs.copy_(hx, non_blocking=True)
            dys.copy_(hdy, non_blocking=True)
        with torch.cuda.stream(ds):
            hdx.copy_(xs, non_blocking=True)
        mlp.forward(x)
        mlp.backward(dy)
    main.wait_stream(cs)
    main.wait_stream(ds)


print("device-only ms/step", timed(dev))
print("device + independent copies ms/step", timed(interfere))
print("device-only again", timed(dev))
