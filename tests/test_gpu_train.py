"""The HQ-FSDP fine-tuning step (BASELINE configs[4]; hqfsdp.hpp:330-414,
trainer.hpp:104-160) on the GPU.

* halo_adamw_step against a host restatement of AdamWT::step (trainer.hpp:
  126-155) in IEEE double with the device's fp32 state storage: bit-exact
  over several steps, bf16 and fp32 masters, bf16 and fp32 gradients.
* HqFsdpLlama (world 1, both data planes -- the library's C++ NCCL plane
  halo_fsdp_* and torch.distributed -- with and without activation
  checkpointing: gathered codes installed per layer, prefetch on a
  side stream, activation checkpointing with one regather feeding the
  recompute and the backward, reduce-scatter, per-layer AdamW) against the
  direct composition -- a stack of block.LlamaBlock's with their own HALO
  layers quantizing W themselves, one autograd graph, no checkpointing, the
  same AdamW -- over two steps: masters, norm gains and dL/dx BIT-IDENTICAL.
  Attention runs on SDPA's deterministic math backend in both.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_02625_b200 import train
    return train


def _bf16_round(a):
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def _adamw_host(w, g, m, v, t, cfg, bf16):
    """AdamWT::step (trainer.hpp:126-155), state stored as fp32."""
    lr_t = cfg.lr * min(1.0, t / cfg.warmup_steps) if cfg.warmup_steps > 0 else cfg.lr
    import math
    bc1 = 1.0 - math.pow(cfg.beta1, float(t))
    bc2 = 1.0 - math.pow(cfg.beta2, float(t))
    gk = g.astype(np.float64)
    mk = cfg.beta1 * m.astype(np.float64) + (1.0 - cfg.beta1) * gk
    vk = cfg.beta2 * v.astype(np.float64) + (1.0 - cfg.beta2) * gk * gk
    mh = mk / bc1
    vh = vk / bc2
    wk = w.astype(np.float64)
    out = (wk - lr_t * (mh / (np.sqrt(vh) + cfg.eps) + cfg.weight_decay * wk)).astype(np.float32)
    if bf16:
        out = _bf16_round(out)
    return out, mk.astype(np.float32), vk.astype(np.float32)


@pytest.mark.parametrize("pdt,gdt", [(torch.bfloat16, torch.float32), (torch.float32, torch.float32),
                                     (torch.bfloat16, torch.bfloat16)])
def test_adamw_matches_reference_formula(T, pdt, gdt):
    n = 1 << 16
    gen = torch.Generator(device="cuda").manual_seed(1)
    p = torch.randn(n, generator=gen, device="cuda").to(pdt)
    cfg = T.AdamWConfig(lr=3e-3, weight_decay=0.01, warmup_steps=2)
    opt = T.DeviceAdamW([p], cfg)
    w = p.float().cpu().numpy()
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    for t in range(1, 5):
        g = (torch.randn(n, generator=gen, device="cuda") * 10 ** (-t)).to(gdt)
        opt.step([g])
        w, m, v = _adamw_host(w, g.float().cpu().numpy(), m, v, t, cfg, pdt == torch.bfloat16)
        torch.cuda.synchronize()
        assert np.array_equal(p.float().cpu().numpy(), w), t
        assert np.array_equal(opt.m[0].cpu().numpy(), m) and np.array_equal(opt.v[0].cpu().numpy(), v), t
    with pytest.raises(ValueError):
        opt.update(0, torch.zeros(n - 4, device="cuda"))


SMALL = dict(hidden=256, heads=2, kv_heads=1, inter=512, layers=2, seq=256)


@pytest.mark.parametrize("plane,ac", [("native", True), ("torch", True), ("native", False)])
def test_fsdp_step_matches_direct_stack(T, plane, ac):
    from torch.nn.attention import SDPBackend, sdpa_kernel

    from paper_2501_02625_b200 import halo
    from paper_2501_02625_b200.block import LlamaBlock
    d = T.LlamaDims(**SMALL)
    scheme = halo.halo2(halo.INT8, 256)
    cfg = T.AdamWConfig(lr=1e-3, warmup_steps=1)
    model = T.HqFsdpLlama(d, scheme, seed=3, opt=cfg, data_plane=plane, activation_checkpoint=ac)
    # the direct composition on copies of the same weights
    blocks = []
    for l in range(d.layers):
        b = LlamaBlock(scheme, hidden=d.hidden, heads=d.heads, kv_heads=d.kv_heads, inter=d.inter, seq=d.seq)
        for name, lin in zip(T.WEIGHTS, b.linears()):
            lin.w.copy_(model.masters[l][name].master)
        blocks.append(b)
    params = []
    for b in blocks:
        params += [lin.w for lin in b.linears()] + [b.n1.data, b.n2.data]
    ref_opt = T.DeviceAdamW(params, cfg)
    tokens = 2 * d.seq
    gen = torch.Generator(device="cuda").manual_seed(11)
    with sdpa_kernel(SDPBackend.MATH):
        for step in range(2):
            x = torch.randn(tokens, d.hidden, generator=gen, device="cuda").to(torch.bfloat16)
            dy = (torch.randn(tokens, d.hidden, generator=gen, device="cuda") * 1e-2).to(torch.bfloat16)
            dx = model.step(x, dy)
            # direct: one graph, no checkpointing, layers quantize their own W
            xin = x.clone().requires_grad_(True)
            h = xin
            for b in blocks:
                for lin in b.linears():
                    lin.grad = None
                b.n1.grad = b.n2.grad = None
                h = b.forward(h)
            h.backward(dy)
            grads = []
            for b in blocks:
                grads += [lin.grad for lin in b.linears()] + [b.n1.grad, b.n2.grad]
            with torch.no_grad():
                ref_opt.step(grads)
            torch.cuda.synchronize()
            assert torch.equal(dx, xin.grad), step
            for l, b in enumerate(blocks):
                for name, lin in zip(T.WEIGHTS, b.linears()):
                    assert torch.equal(model.masters[l][name].master, lin.w), (step, l, name)
                assert torch.equal(model.norms[l][0], b.n1.data) and torch.equal(model.norms[l][1], b.n2.data)
    led = model.ledger
    nw = len(T.WEIGHTS) * d.layers
    assert led.gather.count == 2 * nw * 2          # forward gathers + backward regathers, 2 steps
    assert led.backward_gathers == 2 * nw
    assert led.backward_consumers == 2 * nw * (2 if ac else 1)  # with AC one regather feeds two consumers
    # a master changed after its forward gather (here: by the step's own
    # AdamW update) makes the regather's stale check trip
    model.masters[0]["o"].master.add_(1.0)
    from paper_2501_02625_b200._lib import HaloLogicError
    with pytest.raises(HaloLogicError):
        fsdp_stale(model)


def fsdp_stale(model):
    """regather of layer 0 after its master changed: the device flag trips."""
    from paper_2501_02625_b200 import fsdp
    model.stale.zero_()
    p = model.masters[0]["o"]
    if model.plane is not None:  # the C++ data plane: halo_fsdp_backward_regather's device flag
        model.plane.regather(p, model.rotate, model.block, model.codes[0]["o"], model.ledger, model.stale)
    else:
        fsdp.backward_regather(p, model.rotate, model.ledger, True, model.block, model.group,
                               out=model.codes[0]["o"], stale_flag=model.stale)
    model.check()
