"""Small-shape workload for compute-sanitizer (memcheck / racecheck /
synccheck): K1 (rows FWHT + quantize, both phases), K2 (cols FWHT + dual
quantize), K3 (tcgen05 GEMM, fused K4 epilogue, transposed store), K4,
peer_sync (world 1 mailbox barrier), deq_gemm (row granularity), the glue and
the INT8 split-K path.  Usage: compute-sanitizer --tool X python tools/sanitize_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_2501_02625_b200 import halo  # noqa: E402
from paper_2501_02625_b200._lib import check, lib  # noqa: E402

torch.manual_seed(0)
dev = "cuda"
bf = torch.bfloat16
b, m, n = 256, 512, 256
x = torch.randn(b, m, device=dev).to(bf)
w = (torch.randn(n, m, device=dev) / 16).to(bf)
e = (torch.randn(b, n, device=dev) * 1e-3).to(bf)
for fmt in (halo.INT8, halo.FP8_E4M3):
    for lvl in ("halo0", "halo1", "halo2"):
        layer = halo.HaloLinearLayer(w, halo.scheme_from_string(lvl, fmt, 256), out_dtype=torch.float32)
        ctx = halo.SavedContext()
        layer.forward(x, ctx)
        layer.backward(ctx, e)
        ctx.check()
# row granularity: deq_gemm backward
halo.allow_dequantized_products(True)
layer = halo.HaloLinearLayer(w, halo.halo2(halo.INT8, 256, halo.GRAN_ROW), out_dtype=torch.float32)
ctx = halo.SavedContext()
layer.forward(x, ctx)
layer.backward(ctx, e)
ctx.check()
# standalone K1 / K2 / K4
halo.rotate_quantize(x, 256)
halo.left_rotate_quantize(e, 256)
halo.transform_right(torch.randn(b, m, device=dev), 256)
# INT8 split-K (K > 131072)
K = 131072 + 512
a8 = torch.randint(-127, 128, (K, 128), device=dev, dtype=torch.int8)
b8 = torch.randint(-127, 128, (K, 128), device=dev, dtype=torch.int8)
one = torch.ones(1, device=dev)
halo.qmatmul(a8, b8, one, one, a_kmajor=False, b_kmajor=False)
# glue
g = torch.randn(b, n, device=dev).to(bf)
u = torch.randn(b, n, device=dev).to(bf)
h = torch.empty_like(g)
check(lib().halo_swiglu_forward(halo._ptr(g), halo._ptr(u), halo._ptr(h), g.numel(), halo._stream()))
# peer mailbox barrier, world 1
mb = C.c_void_p()
check(lib().halo_peer_alloc(3 * 4 * 8, C.byref(mb)))
boxes = (C.c_void_p * 1)(mb.value)
am_in = torch.tensor([1.5], device=dev)
am_out = torch.zeros(1, device=dev)
for epoch in (1, 2, 3):
    check(lib().halo_peer_sync(boxes, 1, 0, epoch, halo._ptr(am_in), halo._ptr(am_out), halo._stream()))
torch.cuda.synchronize()
assert am_out.item() == 1.5
check(lib().halo_peer_free(mb))
print("sanitize workload done")
