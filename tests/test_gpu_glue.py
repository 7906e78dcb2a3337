"""Transformer-block glue kernels (llama_glue.cu) on the GPU.

* halo_rmsnorm_forward / _backward in the reference's form (mean = 0, eps =
  0: y = x/||x|| * g) against the UNMODIFIED rmsnorm.hpp:27-100 (oracle/_ref):
  y in fp32 bit-exact for all but a vanishing fraction of elements (the
  device sums x^2 in double in a different order: the double r may differ in
  its last bit, which moves a float rounding only at a near-tie) -- required
  >= 99.99 % identical and max relative error 2^-22; dx (bf16) vs the bf16
  rounding of the reference's fp32 dx within one bf16 ulp; dgain within 1e-6.
* Llama form (mean over dim, eps 1e-5) against a torch fp64 statement.
* RoPE on fused qkv rows against a torch fp32 statement of the rotation
  (same operations, no contraction): bit-exact; backward = transpose.
* The LlamaBlock on these kernels: forward/backward run and stay finite.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_02625_b200 import _lib, block, halo
    return _lib, block, halo


def _norm(L, x, g, mean, eps, out=torch.float32):
    _lib, _, halo = L
    rows, dim = x.shape
    y = torch.empty(rows, dim, dtype=out, device="cuda")
    rstd = torch.empty(rows, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().halo_rmsnorm_forward(halo._ptr(x), halo._ptr(g), halo._ptr(y), halo._dt(y),
                                               halo._ptr(rstd), rows, dim, int(mean), eps, halo._stream()))
    return y, rstd


def _norm_bwd(L, x, dy, g, rstd, mean):
    _lib, _, halo = L
    rows, dim = x.shape
    dx = torch.empty(rows, dim, dtype=torch.bfloat16, device="cuda")
    dg = torch.empty(dim, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().halo_rmsnorm_backward(halo._ptr(x), halo._ptr(dy), halo._dt(dy), halo._ptr(g),
                                                halo._ptr(rstd), halo._ptr(dx), halo._ptr(dg), rows, dim, int(mean),
                                                halo._stream()))
    return dx, dg


@pytest.mark.parametrize("rows,dim", [(64, 256), (37, 4096), (300, 1024)])
def test_rmsnorm_vs_reference(L, orc, rows, dim):
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    g_ = torch.Generator(device="cuda").manual_seed(rows + dim)
    x = torch.randn(rows, dim, generator=g_, device="cuda").to(torch.bfloat16)
    x[:, 5] *= 30
    g = torch.rand(dim, generator=g_, device="cuda") + 0.5
    e = torch.randn(rows, dim, generator=g_, device="cuda").to(torch.bfloat16)
    y, rstd = _norm(L, x, g, mean=False, eps=0.0)
    dx, dg = _norm_bwd(L, x, e, g, rstd, mean=False)
    ry, rdx, rdg = orc.ref_rmsnorm(x.float().cpu().numpy(), g.cpu().numpy(), e.float().cpu().numpy())
    gy = y.cpu().numpy()
    same = float((gy == ry).mean())
    assert same >= 0.9999, same
    assert float(np.max(np.abs(gy - ry) / np.maximum(np.abs(ry), 1e-30))) <= 2.0 ** -22
    want_dx = torch.from_numpy(rdx).to(torch.bfloat16).float().numpy()
    got_dx = dx.float().cpu().numpy()
    ulp = np.abs(want_dx) * 2.0 ** -7 + 1e-30
    assert bool(np.all(np.abs(got_dx - want_dx) <= ulp))
    assert np.allclose(dg.cpu().numpy(), rdg, rtol=1e-6, atol=1e-6)


def test_rmsnorm_llama_form(L):
    _, block, _ = L
    g_ = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(512, 4096, generator=g_, device="cuda").to(torch.bfloat16)
    w = (torch.rand(4096, generator=g_, device="cuda") + 0.5).requires_grad_(True)
    xx = x.clone().requires_grad_(True)
    y = block._rmsnorm(xx, w)
    dy = torch.randn_like(y)
    y.backward(dy)
    xd = x.double().requires_grad_(True)
    wd = w.detach().double().requires_grad_(True)
    yd = xd * torch.rsqrt(xd.pow(2).mean(-1, keepdim=True) + 1e-5) * wd
    yd.backward(dy.double())
    assert torch.equal(y, yd.detach().float().to(torch.bfloat16)) or \
        float(((y.double() - yd.detach()).abs() / yd.detach().abs().clamp_min(1e-30)).max()) <= 2.0 ** -8
    assert float(((xx.grad.double() - xd.grad).abs()).max() / xd.grad.abs().max()) <= 2.0 ** -8
    assert torch.allclose(w.grad.double(), wd.grad, rtol=1e-5, atol=1e-5)


def test_rope_qkv(L):
    _, block, _ = L
    T, seq, nh, nkv, hd = 1024, 512, 4, 2, 128
    cs = block.rope_table(seq, hd, "cuda")
    g_ = torch.Generator(device="cuda").manual_seed(5)
    qkv = torch.randn(T, (nh + 2 * nkv) * hd, generator=g_, device="cuda").to(torch.bfloat16).requires_grad_(True)
    out = block._RopeQKVFn.apply(qkv, cs, seq, nh + nkv, nh + 2 * nkv, hd)
    t = qkv.detach().float().view(T, nh + 2 * nkv, hd)
    pos = torch.arange(T, device="cuda") % seq
    c = cs[pos, :, 0][:, None, :]
    s = cs[pos, :, 1][:, None, :]
    t1, t2 = t[..., : hd // 2], t[..., hd // 2:]
    o = torch.cat((t1 * c - t2 * s, t2 * c + t1 * s), -1)
    o[:, nh + nkv:] = t[:, nh + nkv:]
    assert torch.equal(out, o.reshape(T, -1).to(torch.bfloat16))
    d = torch.randn_like(out)
    out.backward(d)
    dt = d.float().view(T, nh + 2 * nkv, hd)
    d1, d2 = dt[..., : hd // 2], dt[..., hd // 2:]
    want = torch.cat((d1 * c + d2 * s, d2 * c - d1 * s), -1)
    want[:, nh + nkv:] = dt[:, nh + nkv:]
    assert torch.equal(qkv.grad, want.reshape(T, -1).to(torch.bfloat16))


def test_block_on_fused_glue(L):
    _, block, halo = L
    blk = block.LlamaBlock(halo.halo2(halo.INT8, 256), hidden=512, heads=4, kv_heads=2, inter=1024, seq=256)
    x = torch.randn(512, 512, device="cuda").to(torch.bfloat16).requires_grad_(True)
    y = blk.forward(x)
    y.backward(torch.randn_like(y) * 1e-2)
    assert bool(torch.isfinite(y.float()).all()) and bool(torch.isfinite(x.grad.float()).all())
    assert blk.n1.grad is not None and bool(torch.isfinite(blk.n1.grad).all())


@pytest.mark.parametrize("rows,dim", [(300, 512), (1024, 4096)])
def test_add_rmsnorm_matches_unfused(rows, dim):
    """halo_add_rmsnorm_forward / halo_rmsnorm_backward_res (block.py
    _AddRMSNormFn) == torch's bf16 residual add + _RMSNormFn, bit for bit:
    h, the normed output, both input gradients and the gain gradient."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_02625_b200.block import _AddRMSNormFn, _RMSNormFn
    g = torch.Generator(device="cuda").manual_seed(rows)
    bf = torch.bfloat16
    x = torch.randn(rows, dim, generator=g, device="cuda").to(bf)
    r = (torch.randn(rows, dim, generator=g, device="cuda") * 0.3).to(bf)
    w = torch.rand(dim, generator=g, device="cuda") + 0.5
    ch = (torch.randn(rows, dim, generator=g, device="cuda") * 1e-2).to(bf)
    cm = (torch.randn(rows, dim, generator=g, device="cuda") * 1e-2).to(bf)
    outs = []
    for fused in (True, False):
        xi, ri = x.clone().requires_grad_(True), r.clone().requires_grad_(True)
        wi = w.clone().requires_grad_(True)
        if fused:
            h, m = _AddRMSNormFn.apply(xi, ri, wi, 1e-5)
        else:
            h = xi + ri
            m = _RMSNormFn.apply(h, wi, 1e-5)
        ((h * ch).sum() + (m * cm).sum()).backward()
        outs.append((h.detach(), m.detach(), xi.grad, ri.grad, wi.grad))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_rmsnorm_tee_matches_unfused():
    """block.py _RMSNormTeeFn (the first norm of a block, whose input also
    feeds the residual) == _RMSNormFn next to the tensor itself: outputs,
    the input gradient (residual + norm paths) and the gain gradient."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_02625_b200.block import _RMSNormFn, _RMSNormTeeFn
    g = torch.Generator(device="cuda").manual_seed(7)
    bf = torch.bfloat16
    rows, dim = 512, 1024
    x = torch.randn(rows, dim, generator=g, device="cuda").to(bf)
    w = torch.rand(dim, generator=g, device="cuda") + 0.5
    cx = (torch.randn(rows, dim, generator=g, device="cuda") * 1e-2).to(bf)
    ca = (torch.randn(rows, dim, generator=g, device="cuda") * 1e-2).to(bf)
    outs = []
    for fused in (True, False):
        xi, wi = x.clone().requires_grad_(True), w.clone().requires_grad_(True)
        if fused:
            xr, a = _RMSNormTeeFn.apply(xi, wi, 1e-5)
        else:
            xr, a = xi, _RMSNormFn.apply(xi, wi, 1e-5)
        ((xr * cx).sum() + (a * ca).sum()).backward()
        outs.append((a.detach(), xi.grad, wi.grad))
    for p, q in zip(*outs):
        assert torch.equal(p, q)
