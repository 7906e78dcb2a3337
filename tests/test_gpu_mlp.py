"""GPU tests of the Llama MLP block over HALO linears (paper_2501_02625_b200.mlp).

The SwiGLU glue is not part of the reference path; its kernels are checked
against a torch fp32 statement of the same formula (bf16 outputs within a few
ulps: the device sigmoid uses the hardware exp2).  The fused glue
(halo_swiglu_backward_absmax: SwiGLU backward + the absmax pass of both
projections' error quantization) must reproduce the unfused composition
(glue kernel, then two full halo_linear_backward calls) BIT-EXACTLY: same
dG / dU bits, same scales, same codes, hence the same E_X and grad_W.
"""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_02625_b200 import halo, mlp
    return halo, mlp


def _weights(I, H, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    bf = torch.bfloat16
    wg = (torch.randn(I, H, generator=g, device="cuda") / H ** 0.5).to(bf)
    wu = (torch.randn(I, H, generator=g, device="cuda") / H ** 0.5).to(bf)
    wd = (torch.randn(H, I, generator=g, device="cuda") / I ** 0.5).to(bf)
    return wg, wu, wd, g


def test_swiglu_glue_vs_torch(M):
    halo, _ = M
    from paper_2501_02625_b200._lib import check, lib
    g_ = torch.Generator(device="cuda").manual_seed(3)
    n = 1 << 16
    bf = torch.bfloat16
    g = (torch.randn(n, generator=g_, device="cuda") * 3).to(bf)
    u = torch.randn(n, generator=g_, device="cuda").to(bf)
    dh = torch.randn(n, generator=g_, device="cuda").to(bf)
    h = torch.empty_like(g)
    dg = torch.empty_like(g)
    du = torch.empty_like(g)
    check(lib().halo_swiglu_forward(halo._ptr(g), halo._ptr(u), halo._ptr(h), n, halo._stream()))
    check(lib().halo_swiglu_backward(halo._ptr(dh), halo._ptr(g), halo._ptr(u), halo._ptr(dg), halo._ptr(du), n,
                                     halo._stream()))
    gf, uf, dhf = g.float(), u.float(), dh.float()
    s = torch.sigmoid(gf)
    ref_h = gf * s * uf
    ref_du = dhf * gf * s
    ref_dg = dhf * uf * s * (1 + gf * (1 - s))
    for got, ref in ((h, ref_h), (du, ref_du), (dg, ref_dg)):
        err = (got.float() - ref).abs()
        assert bool((err <= 2 ** -6 * ref.abs() + 1e-30).all()), float((err / ref.abs().clamp_min(1e-30)).max())


@pytest.mark.parametrize("fmt", [0, 1])
@pytest.mark.parametrize("T,H,I", [(512, 256, 768), (300, 256, 512), (2048, 512, 1024)])
def test_mlp_fused_glue_bitexact(M, fmt, T, H, I):
    """Fused SwiGLU-backward + K2 absmax == glue kernel + two full backwards."""
    halo, mlp = M
    wg, wu, wd, g = _weights(I, H)
    x = torch.randn(T, H, generator=g, device="cuda").to(torch.bfloat16)
    x[:, [1, 7]] *= 30
    dy = (torch.randn(T, H, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
    outs = []
    for fuse in (False, True):
        m = mlp.HaloMLP(wg, wu, wd, halo.halo2(fmt, 256))
        m.fuse_glue = fuse
        y = m.forward(x)
        dx, grads = m.backward(dy)
        torch.cuda.synchronize()
        outs.append((y.clone(), dx.clone(), [gw.clone() for gw in grads]))
    (y0, dx0, g0), (y1, dx1, g1) = outs
    assert torch.equal(y0, y1)
    assert torch.equal(dx0, dx1)
    for a, b in zip(g0, g1):
        assert torch.equal(a, b)


def test_mlp_fused_glue_other_schemes_fall_back(M):
    """HALO-1 has no left rotation: the fused entry is the plain glue kernel."""
    halo, mlp = M
    wg, wu, wd, g = _weights(512, 256, seed=5)
    x = torch.randn(256, 256, generator=g, device="cuda").to(torch.bfloat16)
    dy = (torch.randn(256, 256, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
    res = []
    for fuse in (False, True):
        m = mlp.HaloMLP(wg, wu, wd, halo.halo1(0, 256))
        m.fuse_glue = fuse
        m.forward(x)
        dx, grads = m.backward(dy)
        torch.cuda.synchronize()
        res.append((dx.clone(), [t.clone() for t in grads]))
    assert torch.equal(res[0][0], res[1][0])
    for a, b in zip(res[0][1], res[1][1]):
        assert torch.equal(a, b)


def test_mlp_stale_absmax_not_reused(M):
    """The precomputed absmax words are consumed only for the same E_Y buffer:
    a backward with a different buffer recomputes them."""
    halo, mlp = M
    wg, wu, wd, g = _weights(512, 256, seed=7)
    x = torch.randn(256, 256, generator=g, device="cuda").to(torch.bfloat16)
    dy = (torch.randn(256, 256, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
    m = mlp.HaloMLP(wg, wu, wd, halo.halo2(0, 256))
    m.forward(x)
    dx1, gr1 = m.backward(dy)
    # same forward context, unfused reference on a fresh module
    r = mlp.HaloMLP(wg, wu, wd, halo.halo2(0, 256))
    r.fuse_glue = False
    r.forward(x)
    dx2, gr2 = r.backward(dy)
    # direct gate backward with another E (copy of dG scaled): must not reuse
    e = (torch.randn(256, 512, generator=g, device="cuda") * 1e-2).to(torch.bfloat16)
    a = m.gate.backward(m.ctx[0], e)
    b = r.gate.backward(r.ctx[0], e)
    torch.cuda.synchronize()
    assert torch.equal(dx1, dx2)
    assert torch.equal(a.e_x, b.e_x)
    assert torch.equal(a.grad_w, b.grad_w)


@pytest.mark.parametrize("fmt", [0, 1, 2])
def test_mlp_fused_forward_glue_bitexact(M, fmt):
    """SwiGLU forward + the down projection's absmax pass in one kernel ==
    glue kernel + the layer's own absmax pass (same h bits, same scale)."""
    halo, mlp = M
    wg, wu, wd, g = _weights(1024, 512, seed=11)
    x = torch.randn(768, 512, generator=g, device="cuda").to(torch.bfloat16)
    x[:, 3] *= 40
    dy = (torch.randn(768, 512, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
    outs = []
    for fuse in (False, True):
        m = mlp.HaloMLP(wg, wu, wd, halo.halo2(fmt, 256))
        m.fuse_fwd = fuse
        y = m.forward(x)
        dx, grads = m.backward(dy)
        torch.cuda.synchronize()
        xq, sx, _, _ = m.ctx[2].saved(m.down)
        outs.append((y.clone(), dx.clone(), [t.clone() for t in grads], xq.clone(), sx.clone()))
    a, b = outs
    assert torch.equal(a[3], b[3]) and torch.equal(a[4], b[4])
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    for u, v in zip(a[2], b[2]):
        assert torch.equal(u, v)


@pytest.mark.parametrize("fmt,b,m,n,gran", [(0, 1000, 512, 768, "tensor"), (1, 777, 256, 512, "tensor"),
                                            (2, 300, 512, 256, "tensor"), (0, 1000, 512, 768, "row"),
                                            (0, 2048, 4096, 14336, "tensor")])
def test_swiglu_epilogue_bitexact(M, fmt, b, m, n, gran):
    """The up projection with h = silu(g) * u in its GEMM epilogue
    (halo_linear_forward_shared_swiglu) == forward_shared + the separate
    halo_swiglu_forward kernel: same u and h bits, ragged token counts
    (rows past b clipped), every format, row granularity, and a cfg2-wide
    (14336-column) projection."""
    halo, _ = M
    from paper_2501_02625_b200._lib import check, lib
    gen = torch.Generator(device="cuda").manual_seed(b + n)
    bf = torch.bfloat16
    scheme = halo.halo2(fmt, 256, halo.GRAN_ROW if gran == "row" else halo.GRAN_TENSOR)
    halo.allow_dequantized_products(gran == "row")  # row-granularity layers (their backward) need the opt-in
    wg = (torch.randn(n, m, generator=gen, device="cuda") / m ** 0.5).to(bf)
    wu = (torch.randn(n, m, generator=gen, device="cuda") / m ** 0.5).to(bf)
    x = torch.randn(b, m, generator=gen, device="cuda").to(bf)
    gate = halo.HaloLinearLayer(wg, scheme, out_dtype=bf)
    up = halo.HaloLinearLayer(wu, scheme, out_dtype=bf)
    cg, c1, c2 = halo.SavedContext(), halo.SavedContext(), halo.SavedContext()
    g = gate.forward(x, cg)
    u_ref = up.forward_shared(cg, c1)
    h_ref = torch.empty_like(g)
    check(lib().halo_swiglu_forward(halo._ptr(g), halo._ptr(u_ref), halo._ptr(h_ref), g.numel(), halo._stream()))
    u, h = up.forward_shared_swiglu(cg, c2, g)
    torch.cuda.synchronize()
    halo.allow_dequantized_products(False)
    assert torch.equal(u, u_ref)
    assert torch.equal(h, h_ref)


@pytest.mark.parametrize("fmt,b", [(0, 1000), (1, 512), (0, 8192)])
def test_residual_epilogue_bitexact(M, fmt, b):
    """HaloMLP.forward(x, residual=r) (the add in the down projection's GEMM
    epilogue, halo_linear_forward_residual) == r + HaloMLP.forward(x) as torch
    adds the two bf16 tensors; ragged and cfg2-sized token counts."""
    halo, mlp = M
    wg, wu, wd, g = _weights(1024, 512, seed=13)
    x = torch.randn(b, 512, generator=g, device="cuda").to(torch.bfloat16)
    r = torch.randn(b, 512, generator=g, device="cuda").to(torch.bfloat16)
    m = mlp.HaloMLP(wg, wu, wd, halo.halo2(fmt, 256))
    y_ref = r + m.forward(x)
    y = m.forward(x, residual=r)
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)


@pytest.mark.parametrize("scheme,b", [("halo2_int8_256", 1000), ("halo2_fp8_128", 512), ("halo2_int8_512", 768),
                                      ("halo1_int8_256", 512)])
def test_backward_acc_bitexact(M, scheme, b):
    """halo_linear_backward_acc (e_x = add + E_X, the add fused into the E
    path's K4 store for HALO-2 blocks <= 256, a separate add otherwise) ==
    halo_linear_backward then a bf16 add; grad_w unchanged."""
    halo, _ = M
    kind, fmt, block = scheme.split("_")
    sch = getattr(halo, kind)(halo.INT8 if fmt == "int8" else halo.FP8_E4M3, int(block))
    g = torch.Generator(device="cuda").manual_seed(b)
    bf = torch.bfloat16
    w = (torch.randn(1024, 512, generator=g, device="cuda") / 512 ** 0.5).to(bf)
    x = torch.randn(b, 512, generator=g, device="cuda").to(bf)
    e = (torch.randn(b, 1024, generator=g, device="cuda") * 1e-2).to(bf)
    a = torch.randn(b, 512, generator=g, device="cuda").to(bf)
    lay = halo.HaloLinearLayer(w, sch, out_dtype=bf)
    ctx = halo.SavedContext()
    lay.forward(x, ctx)
    ref = lay.backward(ctx, e)
    got = lay.backward(ctx, e, e_x_add=a)
    torch.cuda.synchronize()
    assert torch.equal(got.e_x, (a.float() + ref.e_x.float()).to(bf))
    assert torch.equal(got.grad_w, ref.grad_w)


def test_block_fused_glue_matches_unfused(M, monkeypatch):
    """block.attention_block with every glue fusion (tee'd first norm, fused
    residual add + norm, one q/k/v split, the residual add in the down
    projection's epilogue) == the unfused composition: output, input gradient,
    weight and norm-gain gradients bit-identical."""
    halo, _ = M
    from torch.nn.attention import SDPBackend, sdpa_kernel

    from paper_2501_02625_b200 import block
    kw = dict(hidden=512, heads=4, kv_heads=2, inter=1024, seq=256, seed=3)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(512, 512, generator=g, device="cuda").to(torch.bfloat16)
    dy = (torch.randn(512, 512, generator=g, device="cuda") * 1e-2).to(torch.bfloat16)
    outs = []
    with sdpa_kernel(SDPBackend.MATH):
        for unfused in (False, True):
            monkeypatch.setattr(block, "_UNFUSED_GLUE", unfused)
            blk = block.LlamaBlock(halo.halo2(halo.INT8, 256), **kw)
            xi = x.detach().requires_grad_(True)
            y = blk.forward(xi)
            y.backward(dy)
            outs.append([y.detach(), xi.grad] + [l.grad for l in blk.linears()] + [blk.n1.grad, blk.n2.grad])
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_swiglu_epilogue_rejects_unaligned_width(M):
    halo, _ = M
    bf = torch.bfloat16
    gate = halo.HaloLinearLayer(torch.randn(384, 256, device="cuda").to(bf), halo.halo2(0, 256), out_dtype=bf)
    up = halo.HaloLinearLayer(torch.randn(384, 256, device="cuda").to(bf), halo.halo2(0, 256), out_dtype=bf)
    cg = halo.SavedContext()
    g = gate.forward(torch.randn(256, 256, device="cuda").to(bf), cg)
    with pytest.raises(ValueError):
        up.forward_shared_swiglu(cg, halo.SavedContext(), g)


@pytest.mark.parametrize("plane", ["native", "torch"])
def test_fsdp_mlp_world1_matches_mlp(M, plane):
    """FsdpHaloMLP at world 1 (gathers / regathers on a side stream, each
    projection waiting for its own codes, reduce-scatters behind the next
    backward) -- through the library's C++ NCCL data plane or torch.distributed
    -- gives the same bits as the plain HaloMLP."""
    halo, mlp = M
    from paper_2501_02625_b200.fsdp import FsdpHaloMLP
    wg, wu, wd, g = _weights(1024, 512)
    x = torch.randn(512, 512, generator=g, device="cuda").to(torch.bfloat16)
    dy = (torch.randn(512, 512, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
    ref = mlp.HaloMLP(wg, wu, wd, halo.halo2(0, 256))
    f = FsdpHaloMLP(wg, wu, wd, halo.halo2(0, 256), grad_dtype=torch.float32, data_plane=plane, check_stale=True)
    for _ in range(2):
        y0 = ref.forward(x)
        dx0, g0 = ref.backward(dy)
        y1 = f.forward(x)
        dx1, g1 = f.backward(dy)
        torch.cuda.synchronize()
        assert torch.equal(y0, y1) and torch.equal(dx0, dx1)
        for a, b in zip(g0, g1):
            assert torch.equal(a, b)
    assert f.ledger.backward_gathers == 6 and f.ledger.gather.count == 12
    f.close()
