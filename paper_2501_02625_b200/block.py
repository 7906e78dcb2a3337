"""Llama-3 transformer block over HALO linears (cfg3 of BASELINE.json).

    h = x + O( attn( RoPE(QKV(rmsnorm(x))) ) )
    y = h + down( silu(gate(rmsnorm(h))) * up(rmsnorm(h)) )

Every projection is a ``HaloLinearLayer`` (halo_linear.hpp semantics;
HALO-0/1/2, INT8 or FP8-E4M3) wrapped in a torch.autograd.Function, so the
block's backward runs the HALO backward kernels for the projections and
torch autograd for the glue the reference does not cover (RMSNorm, RoPE,
attention via scaled_dot_product_attention); the MLP runs as one
mlp.HaloMLP (the library's SwiGLU and dX-add kernels, gate/up sharing one
quantized X) — the block pattern of
model.hpp:159-209 with the Llama attention added.  ``bf16=True`` builds the
same block on torch.nn.functional.linear (cuBLAS) for the speed-up baseline.
"""
from __future__ import annotations

import os

import torch
import torch.nn.functional as F

from . import halo


class _HaloLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, mod):
        y = mod.layer.forward(x.contiguous(), mod.sctx)
        ctx.mod = mod
        return y

    @staticmethod
    def backward(ctx, dy):
        mod = ctx.mod
        r = mod.layer.backward(mod.sctx, dy.contiguous())
        mod.grad = r.grad_w if mod.grad is None else mod.grad + r.grad_w
        return r.e_x, None


class _HaloMLPFn(torch.autograd.Function):
    """The block's MLP through mlp.HaloMLP: the three HALO projections plus
    the library's SwiGLU / dX-add kernels (one pass each) instead of torch's
    silu / mul / autograd glue."""

    @staticmethod
    def forward(ctx, m, mlp):
        ctx.mlp = mlp
        return mlp.forward(m.contiguous())

    @staticmethod
    def backward(ctx, dy):
        dx, grads = ctx.mlp.backward(dy.contiguous())
        for lin, g in zip(ctx.mlp.owners, grads):  # dW onto the block's gate / up / down
            lin.grad = g if lin.grad is None else lin.grad + g
        return dx, None


class _HaloMLPResFn(torch.autograd.Function):
    """h + MLP(m) with the residual add in the down projection's GEMM
    epilogue (mlp.HaloMLP.forward(m, residual=h)); dh = dy."""

    @staticmethod
    def forward(ctx, m, h, mlp):
        ctx.mlp = mlp
        return mlp.forward(m.contiguous(), residual=h)

    @staticmethod
    def backward(ctx, dy):
        dx, grads = ctx.mlp.backward(dy.contiguous())
        for lin, g in zip(ctx.mlp.owners, grads):
            lin.grad = g if lin.grad is None else lin.grad + g
        return dx, dy, None


class HaloMLPCall:
    """The block's mlp_fn over a HaloMLP: mlp_fn(m) = MLP(m) and, for
    attention_block's residual, mlp_fn(m, h) = h + MLP(m) in one epilogue."""
    residual = True

    def __init__(self, mlp):
        self.mlp = mlp

    def __call__(self, m, h=None):
        if h is None:
            return _HaloMLPFn.apply(m, self.mlp)
        return _HaloMLPResFn.apply(m, h, self.mlp)


class HaloLinear:
    """One projection: weight [out, in] (bf16), a reusable SavedContext."""

    def __init__(self, w: torch.Tensor, scheme, bf16: bool = False):
        # the bf16 reference arm trains the weight too (autograd's dW GEMM),
        # so both arms do the same three GEMMs per projection
        self.w = w.requires_grad_(True) if bf16 else w
        self.bf16 = bf16
        self.grad = None
        if not bf16:
            self.layer = halo.HaloLinearLayer(w, scheme, out_dtype=torch.bfloat16, grad_dtype=torch.float32)
            self.sctx = halo.SavedContext()

    def __call__(self, x):
        if self.bf16:
            return F.linear(x, self.w)
        return _HaloLinearFn.apply(x, self)


def _rmsnorm_torch(x, w, eps=1e-5):
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps) * w).to(x.dtype)


class _RMSNormFn(torch.autograd.Function):
    """Llama RMSNorm on the library kernel (halo_rmsnorm_forward / _backward:
    one pass each; rmsnorm.hpp:27-100 with the 1/dim mean and eps)."""

    @staticmethod
    def forward(ctx, x, w, eps):
        from ._lib import DTYPE_BF16, check, lib
        x = x.contiguous()
        rows, dim = x.shape
        y = torch.empty_like(x)
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
        check(lib().halo_rmsnorm_forward(halo._ptr(x), halo._ptr(w), halo._ptr(y), DTYPE_BF16, halo._ptr(rstd), rows,
                                         dim, 1, eps, halo._stream()))
        ctx.save_for_backward(x, w, rstd)
        return y

    @staticmethod
    def backward(ctx, dy):
        from ._lib import check, lib
        x, w, rstd = ctx.saved_tensors
        dy = dy.contiguous()
        rows, dim = x.shape
        dx = torch.empty_like(x)
        dw = torch.empty(dim, dtype=torch.float32, device=x.device)
        check(lib().halo_rmsnorm_backward(halo._ptr(x), halo._ptr(dy), halo._dt(dy), halo._ptr(w), halo._ptr(rstd),
                                          halo._ptr(dx), halo._ptr(dw), rows, dim, 1, halo._stream()))
        return dx, dw, None


def _rmsnorm(x, w, eps=1e-5):
    return _RMSNormFn.apply(x, w, eps)


class _RMSNormTeeFn(torch.autograd.Function):
    """a = rmsnorm(x) for a block input x that also feeds the residual: the
    Function returns (x, a) so that the residual gradient reaches its backward,
    which folds the autograd engine's bf16 sum dx = RN(dres + rmsnorm'(da))
    into the norm backward's store (halo_rmsnorm_backward_res) instead of a
    separate add.  Bit-identical with `a = _rmsnorm(x)` used next to `x`."""

    @staticmethod
    def forward(ctx, x, w, eps):
        from ._lib import DTYPE_BF16, check, lib
        x = x.contiguous()
        rows, dim = x.shape
        a = torch.empty_like(x)
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
        check(lib().halo_rmsnorm_forward(halo._ptr(x), halo._ptr(w), halo._ptr(a), DTYPE_BF16, halo._ptr(rstd), rows,
                                         dim, 1, eps, halo._stream()))
        ctx.save_for_backward(x, w, rstd)
        return x.view_as(x), a

    @staticmethod
    def backward(ctx, dres, da):
        from ._lib import check, lib
        x, w, rstd = ctx.saved_tensors
        rows, dim = x.shape
        if da is None:
            return dres, None, None
        da = da.contiguous()
        dx = torch.empty_like(x)
        dw = torch.empty(dim, dtype=torch.float32, device=x.device)
        if dres is None:
            check(lib().halo_rmsnorm_backward(halo._ptr(x), halo._ptr(da), halo._dt(da), halo._ptr(w), halo._ptr(rstd),
                                              halo._ptr(dx), halo._ptr(dw), rows, dim, 1, halo._stream()))
        else:
            dres = dres.contiguous()
            check(lib().halo_rmsnorm_backward_res(halo._ptr(x), halo._ptr(da), halo._dt(da), halo._ptr(w),
                                                  halo._ptr(rstd), halo._ptr(dres), halo._ptr(dx), halo._ptr(dw),
                                                  rows, dim, halo._stream()))
        return dx, dw, None


class _AddRMSNormFn(torch.autograd.Function):
    """h = x + r; m = rmsnorm(h) in one kernel (halo_add_rmsnorm_forward),
    and the backward's residual-gradient sum dh + rmsnorm'(dm) fused into the
    norm backward's store (halo_rmsnorm_backward_res).  Bit-identical with
    the unfused torch add + _RMSNormFn: the same bf16 roundings."""

    @staticmethod
    def forward(ctx, x, r, w, eps):
        from ._lib import check, lib
        x, r = x.contiguous(), r.contiguous()
        rows, dim = x.shape
        h = torch.empty_like(x)
        m = torch.empty_like(x)
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
        check(lib().halo_add_rmsnorm_forward(halo._ptr(x), halo._ptr(r), halo._ptr(w), halo._ptr(h), halo._ptr(m),
                                             halo._ptr(rstd), rows, dim, eps, halo._stream()))
        ctx.save_for_backward(h, w, rstd)
        return h, m

    @staticmethod
    def backward(ctx, dh, dm):
        from ._lib import check, lib
        h, w, rstd = ctx.saved_tensors
        rows, dim = h.shape
        if dm is None:
            return dh, dh, None, None
        dm = dm.contiguous()
        dx = torch.empty_like(h)
        dw = torch.empty(dim, dtype=torch.float32, device=h.device)
        if dh is None:
            check(lib().halo_rmsnorm_backward(halo._ptr(h), halo._ptr(dm), halo._dt(dm), halo._ptr(w),
                                              halo._ptr(rstd), halo._ptr(dx), halo._ptr(dw), rows, dim, 1,
                                              halo._stream()))
        else:
            dh = dh.contiguous()
            check(lib().halo_rmsnorm_backward_res(halo._ptr(h), halo._ptr(dm), halo._dt(dm), halo._ptr(w),
                                                  halo._ptr(rstd), halo._ptr(dh), halo._ptr(dx), halo._ptr(dw),
                                                  rows, dim, halo._stream()))
        return dx, dx, dw, None


class _RopeQKVFn(torch.autograd.Function):
    """RoPE on the q and k heads of the fused qkv output (halo_rope_qkv), one
    pass forward and backward."""

    @staticmethod
    def forward(ctx, qkv, cs, seq, rot_heads, heads, hd):
        from ._lib import check, lib
        qkv = qkv.contiguous()
        out = torch.empty_like(qkv)
        check(lib().halo_rope_qkv(halo._ptr(qkv), halo._ptr(out), halo._ptr(cs), qkv.shape[0], seq, rot_heads, heads,
                                  hd, 0, halo._stream()))
        ctx.cs, ctx.args = cs, (seq, rot_heads, heads, hd)
        return out

    @staticmethod
    def backward(ctx, d):
        from ._lib import check, lib
        d = d.contiguous()
        seq, rot_heads, heads, hd = ctx.args
        out = torch.empty_like(d)
        check(lib().halo_rope_qkv(halo._ptr(d), halo._ptr(out), halo._ptr(ctx.cs), d.shape[0], seq, rot_heads, heads,
                                  hd, 1, halo._stream()))
        return out, None, None, None, None, None


def rope_table(seq, hd, device, theta=500000.0):
    """(cos, sin) of pos * inv_freq_i, fp32, [seq, hd/2, 2] (Llama-3 theta)."""
    pos = torch.arange(seq, device=device, dtype=torch.float64)
    inv = 1.0 / (theta ** (torch.arange(0, hd, 2, device=device, dtype=torch.float64) / hd))
    ang = torch.outer(pos, inv)
    return torch.stack((ang.cos(), ang.sin()), -1).float().contiguous()


# HALO_BLOCK_UNFUSED_GLUE=1: the unfused residual add / RMSNorm and q/k/v
# slices (A/B measurements; numerically identical)
_UNFUSED_GLUE = os.environ.get("HALO_BLOCK_UNFUSED_GLUE", "0") == "1"


def attention_block(x, qkv_fn, o_fn, mlp_fn, n1, n2, cs, seq, heads, kv_heads):
    """The Llama block on given projections (shared by LlamaBlock and the
    HQ-FSDP stack, train.HqFsdpLlama):
        h = x + O(attn(RoPE(QKV(rmsnorm(x)))));  y = h + MLP(rmsnorm(h))"""
    T, H = x.shape
    B = T // seq
    hd = H // heads
    if _UNFUSED_GLUE:
        a = _rmsnorm(x, n1)
    else:
        x, a = _RMSNormTeeFn.apply(x, n1, 1e-5)  # x also feeds the residual: its gradient sum is fused
    qkv = _RopeQKVFn.apply(qkv_fn(a), cs, seq, heads + kv_heads, heads + 2 * kv_heads, hd)
    nq, nk = heads * hd, kv_heads * hd
    # one split (its backward is a single cat into dqkv; three slices would
    # each zero-fill a full-size gradient and then sum them)
    if _UNFUSED_GLUE:  # A/B reference: the former slices
        qs, ks, vs = qkv[:, :nq], qkv[:, nq:nq + nk], qkv[:, nq + nk:]
    else:
        qs, ks, vs = qkv.split([nq, nk, nk], dim=1)
    q = qs.view(B, seq, heads, hd).transpose(1, 2)
    k = ks.view(B, seq, kv_heads, hd).transpose(1, 2)
    v = vs.view(B, seq, kv_heads, hd).transpose(1, 2)
    att = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
    att = att.transpose(1, 2).reshape(T, H)
    if _UNFUSED_GLUE:
        h = x + o_fn(att)
        m = _rmsnorm(h, n2)
    else:
        h, m = _AddRMSNormFn.apply(x, o_fn(att), n2, 1e-5)  # h = x + O(att); m = rmsnorm(h)
    if getattr(mlp_fn, "residual", False) and not _UNFUSED_GLUE:
        return mlp_fn(m, h)  # y = h + MLP(m), the add in the down projection's epilogue
    return h + mlp_fn(m)


class LlamaBlock:
    """Llama-3-8B block dims: hidden 4096, 32 query / 8 key-value heads of 128,
    MLP 14336.  Random-init weights (std 1/sqrt(fan_in))."""

    def __init__(self, scheme, hidden=4096, heads=32, kv_heads=8, inter=14336, seq=2048, device="cuda",
                 bf16=False, seed=0):
        g = torch.Generator(device=device).manual_seed(seed)
        bf = torch.bfloat16
        hd = hidden // heads
        self.hidden, self.heads, self.kv, self.hd, self.seq = hidden, heads, kv_heads, hd, seq

        def w(o, i):
            return (torch.randn(o, i, generator=g, device=device) / i ** 0.5).to(bf)

        self.qkv = HaloLinear(w(hidden + 2 * kv_heads * hd, hidden), scheme, bf16)
        self.o = HaloLinear(w(hidden, hidden), scheme, bf16)
        self.gate = HaloLinear(w(inter, hidden), scheme, bf16)
        self.up = HaloLinear(w(inter, hidden), scheme, bf16)
        self.down = HaloLinear(w(hidden, inter), scheme, bf16)
        self.mlp = None
        if not bf16:
            from .mlp import HaloMLP
            self.mlp = HaloMLP(self.gate.w, self.up.w, self.down.w, scheme)
            self.mlp.owners = (self.gate, self.up, self.down)
        self.n1 = torch.ones(hidden, device=device, requires_grad=True)
        self.n2 = torch.ones(hidden, device=device, requires_grad=True)
        self.cs = rope_table(seq, hd, device)

    def linears(self):
        return (self.qkv, self.o, self.gate, self.up, self.down)

    def forward(self, x):
        """x: [batch * seq, hidden] bf16 (requires_grad for the backward)."""
        if self.mlp is not None:
            mlp_fn = HaloMLPCall(self.mlp)
        else:
            mlp_fn = lambda m: self.down(F.silu(self.gate(m)) * self.up(m))  # noqa: E731
        return attention_block(x, self.qkv, self.o, mlp_fn, self.n1, self.n2, self.cs, self.seq, self.heads, self.kv)

    def gemm_ops(self, tokens):
        """6*b*m*n over the five projections (the quantized GEMM work)."""
        return sum(6.0 * tokens * l.w.shape[0] * l.w.shape[1] for l in self.linears())
