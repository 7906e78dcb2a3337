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


class HaloLinear:
    """One projection: weight [out, in] (bf16), a reusable SavedContext."""

    def __init__(self, w: torch.Tensor, scheme, bf16: bool = False):
        self.w = w
        self.bf16 = bf16
        self.grad = None
        if not bf16:
            self.layer = halo.HaloLinearLayer(w, scheme, out_dtype=torch.bfloat16, grad_dtype=torch.float32)
            self.sctx = halo.SavedContext()

    def __call__(self, x):
        if self.bf16:
            return F.linear(x, self.w)
        return _HaloLinearFn.apply(x, self)


def _rmsnorm(x, w, eps=1e-5):
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps) * w).to(x.dtype)


def _rope(t, cos, sin):
    t1, t2 = t[..., : t.shape[-1] // 2], t[..., t.shape[-1] // 2:]
    return torch.cat((t1 * cos - t2 * sin, t2 * cos + t1 * sin), dim=-1)


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
        pos = torch.arange(seq, device=device, dtype=torch.float32)
        inv = 1.0 / (500000.0 ** (torch.arange(0, hd, 2, device=device, dtype=torch.float32) / hd))
        ang = torch.outer(pos, inv)
        self.cos = torch.cat((ang.cos(), ang.cos()), -1).to(bf)[None, None, :, : hd // 2]
        self.sin = torch.cat((ang.sin(), ang.sin()), -1).to(bf)[None, None, :, : hd // 2]

    def linears(self):
        return (self.qkv, self.o, self.gate, self.up, self.down)

    def forward(self, x):
        """x: [batch * seq, hidden] bf16 (requires_grad for the backward)."""
        T, H = x.shape
        B = T // self.seq
        hd, nh, nkv = self.hd, self.heads, self.kv
        a = _rmsnorm(x, self.n1)
        qkv = self.qkv(a)
        q, k, v = qkv.split([nh * hd, nkv * hd, nkv * hd], dim=-1)
        q = q.view(B, self.seq, nh, hd).transpose(1, 2)
        k = k.view(B, self.seq, nkv, hd).transpose(1, 2)
        v = v.view(B, self.seq, nkv, hd).transpose(1, 2)
        q, k = _rope(q, self.cos, self.sin), _rope(k, self.cos, self.sin)
        att = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
        att = att.transpose(1, 2).reshape(T, H)
        h = x + self.o(att)
        m = _rmsnorm(h, self.n2)
        if self.mlp is not None:
            y = h + _HaloMLPFn.apply(m, self.mlp)
        else:
            y = h + self.down(F.silu(self.gate(m)) * self.up(m))
        return y

    def gemm_ops(self, tokens):
        """6*b*m*n over the five projections (the quantized GEMM work)."""
        return sum(6.0 * tokens * l.w.shape[0] * l.w.shape[1] for l in self.linears())
