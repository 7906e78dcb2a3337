"""HQ-FSDP fine-tuning step of a Llama-3-8B decoder stack (BASELINE.json
configs[4]; the reference's train_fsdp loop, hqfsdp.hpp:330-414).

One process per GPU.  Every rank owns a contiguous row shard of each of the
five linear weights of every layer (qkv fused, o, gate, up, down; rows
padded to a multiple of the world size, hqfsdp.hpp:131-148) as a bf16
master, plus AdamW state (trainer.hpp:104-160) for its rows only.  Norm
gains are replicated (hqfsdp.hpp:29).  One step, on this rank's tokens:

  forward   for l = 0..L-1: quantized_all_gather of layer l's (WH)_Q codes
            (hqfsdp.hpp:204-237: K1 absmax of the local shard, absmax
            exchange, K1 quantize under the shared scale, INT8 all-gather),
            issued on a side stream ONE LAYER AHEAD so it overlaps layer
            l-1's GEMMs; the block runs on the gathered codes
            (HaloLinearLayer.set_qweight) without keeping activations: only
            the layer input is saved (activation checkpointing).
  backward  for l = L-1..0: backward_regather under the forward's saved
            scale (hqfsdp.hpp:243-266; stale-weight check), again one layer
            ahead on the side stream; the one regather feeds BOTH consumers,
            the recompute forward and the backward matmuls (hqfsdp.hpp:308-310,
            384: backward_consumers += 2); dW of the five weights is
            reduce-scattered (hqfsdp.hpp:271-300) and the rank's AdamW update
            of its rows runs right away on the device (halo_adamw_step).

The transformer glue (RMSNorm, RoPE, causal GQA attention through
torch.nn.functional.scaled_dot_product_attention) runs in torch autograd;
every projection is a HALO-2 linear (halo_linear.hpp) on the library's
kernels.  Weights are random-initialised (std 1/sqrt(fan_in), model.hpp:
146-149); data is synthetic.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import fsdp, halo
from ._lib import DTYPE_BF16, DTYPE_F32, check, lib
from .block import HaloLinear, HaloMLPCall, attention_block, rope_table


@dataclass
class LlamaDims:
    """Llama-3-8B decoder dims (32 layers, hidden 4096, 32 query / 8 kv heads
    of 128, SwiGLU 14336)."""
    hidden: int = 4096
    heads: int = 32
    kv_heads: int = 8
    inter: int = 14336
    layers: int = 32
    seq: int = 2048

    @property
    def head_dim(self):
        return self.hidden // self.heads

    def shapes(self):
        """(out, in) of the five linear weights of a layer."""
        h, kv = self.hidden, self.kv_heads * self.head_dim
        return {"qkv": (h + 2 * kv, h), "o": (h, h), "gate": (self.inter, h), "up": (self.inter, h),
                "down": (h, self.inter)}


WEIGHTS = ("qkv", "o", "gate", "up", "down")


@dataclass
class AdamWConfig:  # trainer.hpp:95-102
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    warmup_steps: int = 20


class DeviceAdamW:
    """AdamWT (trainer.hpp:104-160) over device tensors: the math runs in the
    library's kernel (IEEE double per element), the state m, v in fp32."""

    def __init__(self, params, cfg: AdamWConfig | None = None):
        self.cfg = cfg or AdamWConfig()
        self.params = list(params)
        self.m = [torch.zeros(p.numel(), dtype=torch.float32, device=p.device) for p in self.params]
        self.v = [torch.zeros(p.numel(), dtype=torch.float32, device=p.device) for p in self.params]
        self.t = 0
        self.lr_t = self.bc1 = self.bc2 = None

    def lr_at(self, step: int) -> float:  # :120-124
        if self.cfg.warmup_steps <= 0:
            return self.cfg.lr
        return self.cfg.lr * min(1.0, float(step) / float(self.cfg.warmup_steps))

    def begin_step(self):  # :126-131
        self.t += 1
        self.lr_t = self.lr_at(self.t)
        self.bc1 = 1.0 - math.pow(self.cfg.beta1, float(self.t))
        self.bc2 = 1.0 - math.pow(self.cfg.beta2, float(self.t))

    def update(self, i: int, grad: torch.Tensor):
        p = self.params[i]
        if grad.numel() != p.numel():
            raise ValueError("adamw: gradient shape mismatch")
        if self.lr_t is None:
            raise RuntimeError("adamw: begin_step() before update()")
        g = grad.contiguous()
        pdt = DTYPE_BF16 if p.dtype == torch.bfloat16 else DTYPE_F32
        gdt = DTYPE_BF16 if g.dtype == torch.bfloat16 else DTYPE_F32
        check(lib().halo_adamw_step(halo._ptr(p), pdt, halo._ptr(g), gdt, halo._ptr(self.m[i]), halo._ptr(self.v[i]),
                                    p.numel(), self.lr_t, self.cfg.beta1, self.cfg.beta2, self.cfg.eps,
                                    self.cfg.weight_decay, self.bc1, self.bc2, halo._stream()))

    def step(self, grads):
        """AdamWT::step: every parameter at once."""
        if len(grads) != len(self.params):
            raise ValueError("adamw: gradient count mismatch")
        self.begin_step()
        for i, g in enumerate(grads):
            self.update(i, g)


class HqFsdpLlama:
    """The cfg5 step: an L-layer Llama-3 decoder whose linear weights live in
    HQ-FSDP shards (see the module docstring)."""

    def __init__(self, dims: LlamaDims, scheme, group=None, seed: int = 0, device="cuda",
                 check_stale: bool = True, prefetch: bool = True, opt: AdamWConfig | None = None,
                 data_plane: str = "native", activation_checkpoint: bool = False):
        self.d = dims
        self.scheme = scheme
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.fmt = scheme.format_w
        self.block = scheme.had_block
        self.rotate = bool(scheme.F.middle)
        # FsdpSimConfig::activation_checkpoint (hqfsdp.hpp:300-310, default
        # off): on, only layer inputs are kept and the backward recomputes
        # each layer on its one regather (two consumers); off, every layer
        # keeps its activations and its own HALO contexts, and the regather
        # feeds the backward alone
        self.ac = activation_checkpoint
        self.check_stale = check_stale
        self.prefetch = prefetch
        self.device = torch.device(device)
        shapes = dims.shapes()
        bf = torch.bfloat16
        # masters: this rank's rows of every weight (identical init on every
        # rank from one seed, then sharded)
        g = torch.Generator(device=self.device).manual_seed(seed)
        wc = fsdp.WorldConfig(self.world)
        self.masters = []
        for _ in range(dims.layers):
            lay = {}
            for name in WEIGHTS:
                o, i = shapes[name]
                w = (torch.randn(o, i, generator=g, device=self.device) / i ** 0.5).to(bf)
                lay[name] = fsdp.shard(w, wc, self.fmt, self.rank)
                del w
            self.masters.append(lay)
        self.norms = [(torch.ones(dims.hidden, device=self.device), torch.ones(dims.hidden, device=self.device))
                      for _ in range(dims.layers)]
        params = []
        for lay, (n1, n2) in zip(self.masters, self.norms):
            params += [lay[name].master for name in WEIGHTS] + [n1, n2]
        self.opt = DeviceAdamW(params, opt)
        # HALO projections run on installed gathered codes (set_qweight); the
        # placeholder weights are never read.  With checkpointing one executor
        # (projections + contexts) and two code slots serve every layer;
        # without, each layer has its own executor and code buffer, since its
        # contexts must live from its forward to its backward
        self._dummy = {name: torch.zeros(shapes[name], dtype=bf, device=self.device) for name in WEIGHTS}
        nexec = 1 if self.ac else dims.layers
        self.execs = [_Executor(self._dummy, scheme) for _ in range(nexec)]
        # without checkpointing every layer keeps its contexts to its
        # backward, but the backwards run one at a time: one backward
        # scratch serves all (≈1.7 GB per layer at 8192 tokens otherwise)
        self._scratch = halo.SavedContext()
        for ex in self.execs:
            for ctx in ex.contexts():
                ctx.share_scratch(self._scratch)
        code_dt = halo.code_dtype(self.fmt)
        p0 = self.masters[0]
        nslots = 2 if self.ac else dims.layers
        self.codes = [{name: torch.empty((p0[name].shard_rows * self.world, p0[name].cols), dtype=code_dt,
                                         device=self.device) for name in WEIGHTS} for _ in range(nslots)]
        self.scales = [dict() for _ in range(nslots)]
        self.comm = torch.cuda.Stream(device=self.device)
        self.ready = [torch.cuda.Event() for _ in range(nslots)]
        self.ledger = fsdp.CommLedger()
        # the collectives: the library's C++ NCCL data plane (halo_fsdp_*) or
        # torch.distributed (the protocol functions of fsdp.py)
        if data_plane not in ("native", "torch"):
            raise ValueError("data_plane: 'native' or 'torch'")
        self.plane = fsdp.NcclDataPlane(group) if data_plane == "native" else None
        self.stale = torch.zeros(1, dtype=torch.int32 if self.plane else torch.float32, device=self.device)
        self.cs = rope_table(dims.seq, dims.head_dim, self.device)

    # ------------------------------------------------------------ weights
    def _slot(self, l: int) -> int:
        return l % 2 if self.ac else l

    def _exec(self, l: int) -> "_Executor":
        return self.execs[0] if self.ac else self.execs[l]

    def _fetch(self, l: int, regather: bool):
        """Gather (or regather) layer l's five code tensors into its slot on
        the side stream; `ready[slot]` fires when they are complete."""
        slot = self._slot(l)
        main = torch.cuda.current_stream(self.device)
        side = self.comm if self.prefetch else main
        # the slot was last read by layer l -/+ 2, enqueued before this point
        side.wait_stream(main)
        with torch.cuda.stream(side):
            for name in WEIGHTS:
                p = self.masters[l][name]
                out = self.codes[slot][name]
                if regather:
                    if self.plane is not None:
                        codes, scale = self.plane.regather(p, self.rotate, self.block, out, self.ledger,
                                                           self.stale if self.check_stale else None)
                    else:
                        codes, scale = fsdp.backward_regather(p, self.rotate, self.ledger, self.check_stale,
                                                              self.block, self.group, out=out, stale_flag=self.stale)
                    # with checkpointing one regather feeds two consumers:
                    # the recompute forward and the backward (:308-310, 384)
                    self.ledger.backward_consumers += 2 if self.ac else 1
                elif self.plane is not None:
                    codes, scale = self.plane.gather(p, self.rotate, self.block, out, self.ledger)
                else:
                    codes, scale = fsdp.quantized_all_gather(p, self.rotate, self.ledger, self.block, self.group,
                                                             out=out)
                self.scales[slot][name] = scale
            self.ready[slot].record(side)

    def _install(self, l: int, wait: bool = True):
        slot = self._slot(l)
        if wait:
            torch.cuda.current_stream(self.device).wait_event(self.ready[slot])
        ex = self._exec(l)
        for name in WEIGHTS:
            p = self.masters[l][name]
            ex.layers_of[name].set_qweight(self.codes[slot][name][: p.full_rows], self.scales[slot][name])

    # -------------------------------------------------------------- block
    def _block(self, x: torch.Tensor, l: int) -> torch.Tensor:
        """Llama block (block.attention_block) on the installed codes."""
        d = self.d
        n1, n2 = self.norms[l]
        ex = self._exec(l)
        return attention_block(x, ex.lin["qkv"], ex.lin["o"], HaloMLPCall(ex.mlp), n1, n2,
                               self.cs, d.seq, d.heads, d.kv_heads)

    # --------------------------------------------------------------- step
    def step(self, x: torch.Tensor, dy: torch.Tensor) -> torch.Tensor:
        """One fine-tuning step on this rank's tokens x [T, hidden] (T a
        multiple of seq) with upstream gradient dy at the stack output.
        Returns dL/dx of the stack input."""
        L = self.d.layers
        self.opt.begin_step()
        # ---------------- forward (weights gathered one layer ahead)
        saved = []
        h = x
        self._fetch(0, regather=False)
        for l in range(L):
            self._install(l)
            if l + 1 < L:
                self._fetch(l + 1, regather=False)
            if self.ac:  # only the layer input is kept
                with torch.no_grad():
                    saved.append(h)
                    h = self._block(h, l)
            else:  # the layer's graph (and its HALO contexts) live until its backward
                n1, n2 = self.norms[l]
                n1.requires_grad_(True)
                n2.requires_grad_(True)
                xin = h.detach().requires_grad_(True)
                with torch.enable_grad():
                    y = self._block(xin, l)
                saved.append((xin, y))
                h = y.detach()
        # ---------------- backward (regathered one layer ahead)
        g = dy
        self.stale.zero_()
        self._fetch(L - 1, regather=True)
        for l in reversed(range(L)):
            if self.ac:
                self._install(l)  # the recompute forward and the backward read the regathered codes
            else:
                # the contexts saved at the forward point at this layer's
                # buffer, which the regather rewrote in place
                torch.cuda.current_stream(self.device).wait_event(self.ready[self._slot(l)])
            if l > 0:
                self._fetch(l - 1, regather=True)
            ex = self._exec(l)
            ex.zero_grads()
            n1, n2 = self.norms[l]
            if self.ac:
                n1.grad = n2.grad = None
                n1.requires_grad_(True)
                n2.requires_grad_(True)
                xin = saved[l].detach().requires_grad_(True)
                with torch.enable_grad():
                    y = self._block(xin, l)  # recompute on the same regathered codes
            else:
                xin, y = saved[l]
            y.backward(g)
            g = xin.grad
            saved[l] = None
            grads = ex.grads()
            base = l * (len(WEIGHTS) + 2)
            for j, name in enumerate(WEIGHTS):
                p = self.masters[l][name]
                if self.plane is not None:
                    gshard = self.plane.reduce_scatter(grads[name], p, self.ledger)
                else:
                    gshard = fsdp.reduce_scatter_grads(grads[name], p, self.ledger, self.group)
                self.opt.update(base + j, gshard)
            for j, n in enumerate((n1, n2)):
                ng = n.grad
                if self.world > 1:
                    if self.plane is not None:
                        self.plane.all_reduce_mean(ng)
                    else:
                        dist.all_reduce(ng, group=self.group)
                        ng.div_(self.world)
                n.requires_grad_(False)
                self.opt.update(base + len(WEIGHTS) + j, ng)
                n.grad = None
            ex.zero_grads()
        if self.check_stale:
            torch.cuda.current_stream(self.device).wait_stream(self.comm)
            fsdp.check_stale_flag(self.stale, self.group)
        return g

    def check(self):
        """Synchronise and raise on the step's device-side stale flag."""
        fsdp.check_stale_flag(self.stale, self.group)

    def gemm_ops(self, tokens: int) -> float:
        """6*b*m*n of the five projections per layer (the quantized GEMM work),
        plus the recompute forward's 2*b*m*n under activation checkpointing."""
        per = sum(o * i for o, i in self.d.shapes().values())
        return (8.0 if self.ac else 6.0) * tokens * per * self.d.layers

    def close(self):
        torch.cuda.synchronize(self.device)
        if self.plane is not None:
            self.plane.close()


class _GradSink:
    """dW accumulator for a projection of the shared MLP (block._HaloMLPFn)."""

    def __init__(self):
        self.grad = None


class _Executor:
    """The five HALO projections of one Llama layer (qkv and o as
    block.HaloLinear, gate / up / down as one HaloMLP) on placeholder weights;
    gathered codes are installed per layer."""

    def __init__(self, dummy, scheme):
        from .mlp import HaloMLP
        self.lin = {name: HaloLinear(dummy[name], scheme) for name in ("qkv", "o")}
        self.mlp = HaloMLP(dummy["gate"], dummy["up"], dummy["down"], scheme)
        self.owners = [_GradSink(), _GradSink(), _GradSink()]
        self.mlp.owners = self.owners
        self.layers_of = {"qkv": self.lin["qkv"].layer, "o": self.lin["o"].layer, "gate": self.mlp.gate,
                          "up": self.mlp.up, "down": self.mlp.down}

    def contexts(self):
        return [self.lin["qkv"].sctx, self.lin["o"].sctx] + list(self.mlp.ctx)

    def zero_grads(self):
        for lin in self.lin.values():
            lin.grad = None
        for s in self.owners:
            s.grad = None

    def grads(self):
        return {"qkv": self.lin["qkv"].grad, "o": self.lin["o"].grad, "gate": self.owners[0].grad,
                "up": self.owners[1].grad, "down": self.owners[2].grad}
