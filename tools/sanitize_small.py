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

# ---- round-2 kernels: large-block K1/K4, MX quantizer + MXFP6 layer, RMSNorm,
# RoPE, AdamW, FP6 wire format, the NCCL data plane at world 1
for blk in (512, 4096):
    xl = torch.randn(8, 8192, device=dev).to(bf)
    halo.rotate_quantize(xl, blk)
    halo.transform_right(torch.randn(8, 8192, device=dev), blk)
halo.rotate_quantize_mx(x, 256)
halo.rotate_quantize_mx(e, transpose=True)
mxl = halo.HaloLinearLayer(w, halo.halo2(halo.MXFP6_E3M2, 256, halo.GRAN_MX), out_dtype=torch.float32)
ctx = halo.SavedContext()
mxl.forward(x, ctx)
mxl.backward(ctx, e)
ctx.check()
from paper_2501_02625_b200 import block  # noqa: E402
xn = torch.randn(64, 512, device=dev).to(bf).requires_grad_(True)
wn = torch.ones(512, device=dev, requires_grad=True)
yn = block._rmsnorm(xn, wn)
yn.backward(torch.randn_like(yn))
qkv = torch.randn(256, 4 * 128, device=dev).to(bf).requires_grad_(True)
ro = block._RopeQKVFn.apply(qkv, block.rope_table(128, 128, dev), 128, 3, 4, 128)
ro.backward(torch.randn_like(ro))
from paper_2501_02625_b200.train import DeviceAdamW  # noqa: E402
pw = torch.randn(4096, device=dev).to(bf)
opt = DeviceAdamW([pw])
opt.step([torch.randn(4096, device=dev)])
c6, _ = halo.rotate_quantize(x, 256, fmt=halo.FP6_E3M2)
halo.fp6_unpack(halo.fp6_pack(c6), c6.numel())
from paper_2501_02625_b200.fsdp import FsdpHaloMLP  # noqa: E402
wg_ = (torch.randn(512, 256, device=dev) / 16).to(bf)
wd_ = (torch.randn(256, 512, device=dev) / 16).to(bf)
f = FsdpHaloMLP(wg_, wg_.clone(), wd_, halo.halo2(halo.INT8, 256), check_stale=True)
f.forward(torch.randn(256, 256, device=dev).to(bf))
f.backward(torch.randn(256, 256, device=dev).to(bf) * 1e-3)
f.close()
# large-block left transform (fwht_cols_lb.cu): bf16 / fp32, padded token block, transform-only
for B in (512, 1024, 2048, 4096):
    el = (torch.randn(B - 37, 16384 // B * 2 if B < 4096 else 16, device=dev) * 1e-3)
    halo.left_rotate_quantize(el.to(bf), B)
    halo.left_rotate_quantize(el, B)
    halo.transform_left(torch.randn(B, max(8, 16384 // B), device=dev), B)
# fused residual add + RMSNorm (block.py _AddRMSNormFn)
xa = torch.randn(64, 512, device=dev).to(bf).requires_grad_(True)
ra = torch.randn(64, 512, device=dev).to(bf).requires_grad_(True)
ha, ma = block._AddRMSNormFn.apply(xa, ra, torch.ones(512, device=dev, requires_grad=True), 1e-5)
((ha * 0.5).sum() + ma.sum()).backward()
# SwiGLU GEMM epilogue (halo_linear_forward_shared_swiglu): ragged token count
wgs = (torch.randn(512, 256, device=dev) / 16).to(bf)
gate_s = halo.HaloLinearLayer(wgs, halo.halo2(halo.INT8, 256), out_dtype=bf)
up_s = halo.HaloLinearLayer(wgs.clone(), halo.halo2(halo.INT8, 256), out_dtype=bf)
cgs = halo.SavedContext()
gs = gate_s.forward(torch.randn(300, 256, device=dev).to(bf), cgs)
up_s.forward_shared_swiglu(cgs, halo.SavedContext(), gs)
# residual epilogue (halo_linear_forward_residual): ragged token count
dn_s = halo.HaloLinearLayer((torch.randn(256, 512, device=dev) / 16).to(bf), halo.halo2(halo.INT8, 256), out_dtype=bf)
dn_s.forward_residual(gs, halo.SavedContext(), torch.randn(300, 256, device=dev).to(bf))
# dX accumulated into the K4 store (halo_linear_backward_acc), ragged tokens
cac = halo.SavedContext()
la = halo.HaloLinearLayer((torch.randn(512, 256, device=dev) / 16).to(bf), halo.halo2(halo.INT8, 256), out_dtype=bf)
la.forward(torch.randn(300, 256, device=dev).to(bf), cac)
la.backward(cac, torch.randn(300, 512, device=dev).to(bf) * 1e-2, e_x_add=torch.randn(300, 256, device=dev).to(bf))
# the block's first norm with the residual-gradient sum (block.py _RMSNormTeeFn)
xt_ = torch.randn(64, 512, device=dev).to(bf).requires_grad_(True)
xr_, at_ = block._RMSNormTeeFn.apply(xt_, torch.ones(512, device=dev, requires_grad=True), 1e-5)
((xr_ * 0.5).sum() + at_.sum()).backward()
torch.cuda.synchronize()
print("sanitize workload (round-2 kernels) done")
