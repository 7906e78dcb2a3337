"""Llama-3 MLP block over three HALO linears (cfg2 of BASELINE.json).

    y = down( silu(gate(x)) * up(x) )

The three projections are ``HaloLinearLayer`` instances (halo_linear.hpp
semantics, HALO-0/1/2, INT8 or FP8); the SwiGLU glue and the residual-style
add of the two input gradients are sm_100a kernels of the same library.
This is the reference's block pattern (model.hpp:159-176: norm -> fc1 ->
silu -> fc2, backward in reverse :179-209) with the Llama gate added.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from . import halo
from ._lib import DTYPE_BF16, check, lib


class HaloMLP:
    def __init__(self, w_gate: torch.Tensor, w_up: torch.Tensor, w_down: torch.Tensor, scheme):
        hidden, model = w_gate.shape
        if tuple(w_up.shape) != (hidden, model) or tuple(w_down.shape) != (model, hidden):
            raise ValueError("HaloMLP: weight shapes must be gate/up (I x H) and down (H x I)")
        bf = torch.bfloat16
        self.gate = halo.HaloLinearLayer(w_gate, scheme, out_dtype=bf)
        self.up = halo.HaloLinearLayer(w_up, scheme, out_dtype=bf)
        self.down = halo.HaloLinearLayer(w_down, scheme, out_dtype=bf)
        self.ctx = [halo.SavedContext() for _ in range(3)]
        self._act = None
        self.share_x = True
        # SwiGLU backward fused with the absmax pass of the gate/up error
        # quantization (halo_swiglu_backward_absmax); False = separate kernels
        self.fuse_glue = os.environ.get("HALO_MLP_FUSE_GLUE", "0") == "1"
        # SwiGLU forward fused with the down projection's absmax pass
        # (halo_swiglu_forward_absmax, bit-exact; off: measured slower, see DESIGN)
        self.fuse_fwd = os.environ.get("HALO_MLP_FUSE_FWD", "0") == "1"
        # SwiGLU product in the up projection's GEMM epilogue (bit-identical;
        # HALO_MLP_GLU_EPI=0: the separate halo_swiglu_forward kernel)
        self.glu_epi = os.environ.get("HALO_MLP_GLU_EPI", "1") == "1" and hidden % 256 == 0
        # forward(x, residual): the add in the down projection's GEMM epilogue
        # (bit-identical; HALO_MLP_RES_EPI=0: a separate bf16 add)
        self.res_epi = os.environ.get("HALO_MLP_RES_EPI", "1") == "1"
        # dx = ex_gate + ex_up fused into the up projection's K4 store
        # (halo_linear_backward_acc, bit-identical; HALO_MLP_ACC_DX=0: halo_add)
        self.acc_dx = os.environ.get("HALO_MLP_ACC_DX", "1") == "1"
        # tests: a dict here collects the step's intermediate tensors
        self.trace = None
        # HQ-FSDP hooks: pre(name, phase) runs before a projection's GEMMs
        # (waits for its gathered codes), post_grad(name, grad_w) right after
        # its backward (launches its reduce-scatter)
        self.pre = None
        self.post_grad = None

    def _pre(self, name, phase):
        if self.pre is not None:
            self.pre(name, phase)

    def _post(self, name, grad):
        if self.post_grad is not None:
            return self.post_grad(name, grad)
        return grad

    def forward(self, x: torch.Tensor, residual: torch.Tensor = None) -> torch.Tensor:
        """y = down(silu(gate(x)) * up(x)), plus ``residual`` when given (the
        block's y = h + MLP(.), added in the down projection's GEMM epilogue)."""
        self._pre("gate", "fwd")
        g = self.gate.forward(x, self.ctx[0])
        # up_proj sees the same X under the same quantizer: reuse gate's (XH)_Q
        self._pre("up", "fwd")
        if self.share_x and self.glu_epi and not self.fuse_fwd:
            # h = silu(g) * u computed in the up projection's GEMM epilogue
            u, h = self.up.forward_shared_swiglu(self.ctx[0], self.ctx[1], g)
        else:
            u = self.up.forward_shared(self.ctx[0], self.ctx[1]) if self.share_x else self.up.forward(x, self.ctx[1])
            h = torch.empty_like(g)
            if self.fuse_fwd:
                # SwiGLU + the down projection's absmax pass in one read of g, u
                check(lib().halo_swiglu_forward_absmax(self.down._h, self.ctx[2]._h, halo._ptr(g), halo._ptr(u),
                                                       halo._ptr(h), g.shape[0], g.shape[1], halo._stream()))
            else:
                check(lib().halo_swiglu_forward(halo._ptr(g), halo._ptr(u), halo._ptr(h), g.numel(), halo._stream()))
        self._act = (g, u)
        self._pre("down", "fwd")
        if residual is None:
            y = self.down.forward(h, self.ctx[2])
        elif self.res_epi and self.down.out_features % 256 == 0 and self.down.out_dtype == torch.bfloat16:
            y = self.down.forward_residual(h, self.ctx[2], residual.contiguous())
        else:
            y = residual + self.down.forward(h, self.ctx[2])
        if self.trace is not None:
            self.trace.update(g=g, u=u, h=h, y=y)
        return y

    def backward(self, dy: torch.Tensor, need_grad_w: bool = True):
        """Returns (dx, (dW_gate, dW_up, dW_down))."""
        g, u = self._act
        self._pre("down", "bwd")
        bd = self.down.backward(self.ctx[2], dy, need_grad_w)
        gd = self._post("down", bd.grad_w)
        dg = torch.empty_like(g)
        du = torch.empty_like(u)
        if self.fuse_glue:
            check(lib().halo_swiglu_backward_absmax(self.gate._h, self.ctx[0]._h, self.up._h, self.ctx[1]._h,
                                                    halo._ptr(bd.e_x), halo._ptr(g), halo._ptr(u), halo._ptr(dg),
                                                    halo._ptr(du), g.shape[0], g.shape[1], halo._stream()))
        else:
            check(lib().halo_swiglu_backward(halo._ptr(bd.e_x), halo._ptr(g), halo._ptr(u), halo._ptr(dg),
                                             halo._ptr(du), g.numel(), halo._stream()))
        self._pre("gate", "bwd")
        bg = self.gate.backward(self.ctx[0], dg, need_grad_w)
        gg = self._post("gate", bg.grad_w)
        self._pre("up", "bwd")
        if self.trace is None and self.acc_dx:
            # dx = ex_gate + ex_up, the add fused into up's K4 store
            bu = self.up.backward(self.ctx[1], du, need_grad_w, e_x_add=bg.e_x)
            dx = bu.e_x
        else:
            bu = self.up.backward(self.ctx[1], du, need_grad_w)
            dx = torch.empty_like(bg.e_x)
            check(lib().halo_add(halo._ptr(bg.e_x), halo._ptr(bu.e_x), halo._ptr(dx), DTYPE_BF16, dx.numel(),
                                 halo._stream()))
        gu = self._post("up", bu.grad_w)
        if self.trace is not None:
            self.trace.update(dh=bd.e_x, dg=dg, du=du, ex_gate=bg.e_x, ex_up=bu.e_x)
        return dx, (gg, gu, gd)

    def gemm_ops(self, tokens: int) -> float:
        """Integer ops of the three quantized GEMM triples: 6*b*m*n each."""
        ops = 0.0
        for l in (self.gate, self.up, self.down):
            ops += 6.0 * tokens * l.in_features * l.out_features
        return ops


def profile_enable(on: bool = True):
    check(lib().halo_profile_enable(1 if on else 0))


def profile_read() -> dict:
    from ._lib import Profile
    p = Profile()
    check(lib().halo_profile_read(C.byref(p)))
    return p.as_dict()
