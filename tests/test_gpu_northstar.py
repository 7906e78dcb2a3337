"""Parity at the north_star shapes (BASELINE.json configs[0] and [1]).

cfg1: HALO-2 INT8, b=2048 tokens, 4096 -> 4096, Hadamard block 256.
cfg2: the Llama-3-8B MLP projections at 8192 tokens: gate/up 4096 -> 14336
and down 14336 -> 4096, INT8 and FP8 E4M3, block 256; plus one HaloMLP step
checked projection by projection.

The oracle's naive layer (orc.linear) is far too slow at these sizes, so every
stage is checked on its own, against the C restatement (oracle/halo_oracle.c)
where it is cheap and against exact arithmetic where it is not:

* K1 / K2 codes and scales: byte-exact vs orc.quantize(orc.fwht_rows / cols)
  (quantize.hpp:244-280, hadamard.hpp:136-216) on the same bf16 inputs.
* K3 accumulators: exact.  The codes (already proven equal to the oracle's)
  are multiplied in float64 on the GPU: INT8 products are integers and
  |acc| <= K*127^2 < 2^53, E4M3 products carry 8 significant bits over
  2^-18..2^17.6, so every partial sum is exact in any order.
* The epilogue: float(double(acc) * (double(sa) * double(sb)))
  (quantize.hpp:356-370) evaluated in torch float64 (IEEE, RNE to float).
* The output transforms: orc.fwht_cols (transform_left, :405-409) and
  orc.fwht_rows (transform_right_ht, :410-411, :436-437) on the host.

Tolerances: INT8 0 (bit-exact fp32; bf16 outputs = RNE of the fp32 values).
FP8 E4M3: codes / scales bit-exact; outputs within 1e-5 relative (Frobenius)
of the reference's dequantized double products (the tensor core accumulates
in fp32).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

BLOCK = 256
FP8_TOL = 1e-5


@pytest.fixture(scope="module")
def H():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_02625_b200 import halo
    return halo


def _inputs(b, m, n, seed):
    """SURVEY §8d data on the device: X ~ N(0,1) with outlier columns x40,
    W ~ N(0, 1/sqrt(m)) with outlier columns x20, E_Y ~ N(0, 1e-3) with two
    outlier token rows x30; all bf16."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(b, m, generator=g, device="cuda")
    x[:, [2, 9, 16, 27]] *= 40
    w = torch.randn(n, m, generator=g, device="cuda") / m ** 0.5
    w[:, [5, 19]] *= 20
    e = torch.randn(b, n, generator=g, device="cuda") * 1e-3
    e[[3, b // 2], :] *= 30
    bf = torch.bfloat16
    return x.to(bf), w.to(bf), e.to(bf)


def _np(t):
    return t.float().cpu().numpy()


def _code_values(codes, fmt):
    if fmt == 0:
        return codes.view(torch.int8).double()
    return codes.view(torch.float8_e4m3fn).double()


def _exact_acc(a, b, fmt):
    """acc[i, j] = sum_k a[i, k] * b[k, j] over code values, exact (float64)."""
    return _code_values(a, fmt) @ _code_values(b, fmt)


def _epilogue(acc, sa, sb):
    """float(double(acc) * (double(sa) * double(sb)))  (quantize.hpp:356-370)"""
    return (acc * (sa.double() * sb.double())).float()


def _assert_codes(orc, got_codes, got_scale, want_vals, fmt, what):
    want_codes, want_s = orc.quantize(want_vals, fmt)
    assert got_scale.item() == want_s[0], f"{what}: scale {got_scale.item()!r} != {want_s[0]!r}"
    got = got_codes.cpu().numpy().view(np.uint8)
    want = orc.codes_to_bytes(want_codes, fmt).view(np.uint8)
    assert got.shape == want.shape
    bad = int((got != want).sum())
    assert bad == 0, f"{what}: {bad} of {got.size} codes differ"


def _assert_out(got, want_f32, fmt, what):
    """got: device tensor (fp32 or bf16); want_f32: numpy fp32 oracle."""
    if fmt == 0:
        want = torch.from_numpy(np.ascontiguousarray(want_f32))
        if got.dtype == torch.bfloat16:
            want = want.to(torch.bfloat16)
        g = got.cpu()
        bad = int((g.view(torch.int16 if g.dtype == torch.bfloat16 else torch.int32) !=
                   want.view(torch.int16 if want.dtype == torch.bfloat16 else torch.int32)).sum())
        assert bad == 0, f"{what}: {bad} of {g.numel()} values differ from the oracle"
    else:
        g = got.float().cpu().numpy().astype(np.float64)
        w = want_f32.astype(np.float64)
        r = np.linalg.norm(g - w) / max(np.linalg.norm(w), 1e-300)
        assert r <= FP8_TOL, f"{what}: relative error {r:.3e} > {FP8_TOL}"


def check_forward(orc, fmt, x_np, w_np, xq, sx, wq, sw, y, rotate=True):
    """(XH)_Q, (WH)_Q and Y = qmatmul(xq, wq^T) (halo_linear.hpp:292-299)."""
    xr = orc.fwht_rows(x_np, BLOCK) if rotate else x_np
    _assert_codes(orc, xq, sx, xr, fmt, "xq")
    del xr
    wr = orc.fwht_rows(w_np, BLOCK) if rotate else w_np
    _assert_codes(orc, wq, sw, wr, fmt, "wq")
    del wr
    acc = _exact_acc(xq, wq.t(), fmt)
    want = _epilogue(acc, sx, sw)
    del acc
    _assert_out(y, want.cpu().numpy(), fmt, "Y")


def check_backward(orc, fmt, e_np, xq, sx, wq, sw, ops, e_x, grad_w):
    """HALO-2 error and gradient paths (halo_linear.hpp:381-439):
    E_X = H_b^T (H_b E_Y)_Q (WH)_Q H_m^T,  G = (E_Y^T)_Q (XH)_Q H_m^T."""
    b, n = e_np.shape
    bp = ops["ehq"].shape[0]
    pad = np.zeros((bp, n), np.float32)
    pad[:b] = e_np
    _assert_codes(orc, ops["ehq"], ops["seh"], orc.fwht_cols(pad, BLOCK), fmt, "(H_b E_Y)_Q")
    del pad
    _assert_codes(orc, ops["eq"], ops["se"], e_np, fmt, "(E_Y)_Q")
    # E: prod = qmatmul(ehq, wq) -> transform_left -> take_rows(b) -> transform_right_ht
    acc = _exact_acc(ops["ehq"], wq, fmt)
    P = _epilogue(acc, ops["seh"], sw).cpu().numpy()
    del acc
    P = orc.fwht_cols(P, BLOCK)[:b]
    P = orc.fwht_rows(np.ascontiguousarray(P), BLOCK)
    _assert_out(e_x, P, fmt, "E_X")
    del P
    # G: qmatmul(transpose_quantized(eq), xq) -> transform_right_ht
    if grad_w is not None:
        acc = _exact_acc(ops["eq"].t(), xq, fmt)
        G = _epilogue(acc, ops["se"], sx).cpu().numpy()
        del acc
        G = orc.fwht_rows(G, BLOCK)
        _assert_out(grad_w, G, fmt, "grad_W")


SHAPES = {
    "cfg1": (2048, 4096, 4096),
    "cfg2_gate_up": (8192, 4096, 14336),
    "cfg2_down": (8192, 14336, 4096),
}


@pytest.mark.parametrize("shape,fmt", [("cfg1", 0), ("cfg2_gate_up", 0), ("cfg2_down", 0),
                                       ("cfg2_gate_up", 1), ("cfg2_down", 1)])
def test_layer_at_northstar_shape(H, orc, shape, fmt):
    b, m, n = SHAPES[shape]
    x, w, e = _inputs(b, m, n, seed=17 + b + m)
    layer = H.HaloLinearLayer(w, H.halo2(fmt, BLOCK), out_dtype=torch.float32)
    ctx = H.SavedContext()
    y = layer.forward(x, ctx)
    back = layer.backward(ctx, e)
    ctx.check()
    xq, sx, wq, sw = ctx.saved(layer)
    ops = ctx.error_operands(layer)
    torch.cuda.synchronize()
    x_np, w_np, e_np = _np(x), _np(w), _np(e)
    check_forward(orc, fmt, x_np, w_np, xq, sx, wq, sw, y)
    del y
    check_backward(orc, fmt, e_np, xq, sx, wq, sw, ops, back.e_x, back.grad_w)
    c = layer.counters()
    assert (c.x, c.w, c.e) == (1, 1, 2)


def test_mlp_step_at_cfg2(H, orc):
    """One HaloMLP fwd+bwd at cfg2 (8192 tokens, 4096 -> 14336 -> 4096, HALO-2
    INT8, block 256), every projection checked bit-exactly with the stages
    above on the tensors the step actually fed it; the SwiGLU glue against a
    torch fp32 statement of the formula (not on the reference path)."""
    from paper_2501_02625_b200 import mlp as M
    from paper_2501_02625_b200._lib import check, lib
    T, Hd, I = 8192, 4096, 14336
    g_ = torch.Generator(device="cuda").manual_seed(5)
    bf = torch.bfloat16
    wg = (torch.randn(I, Hd, generator=g_, device="cuda") / Hd ** 0.5).to(bf)
    wu = (torch.randn(I, Hd, generator=g_, device="cuda") / Hd ** 0.5).to(bf)
    wd = (torch.randn(Hd, I, generator=g_, device="cuda") / I ** 0.5).to(bf)
    x = torch.randn(T, Hd, generator=g_, device="cuda")
    x[:, [2, 9, 16, 27]] *= 40
    x = x.to(bf)
    dy = (torch.randn(T, Hd, generator=g_, device="cuda") * 1e-3).to(bf)
    mlp = M.HaloMLP(wg, wu, wd, H.halo2(0, BLOCK))
    mlp.trace = {}
    mlp.forward(x)
    dx, (gw_g, gw_u, gw_d) = mlp.backward(dy)
    for c in mlp.ctx:
        c.check()
    t = mlp.trace
    g, u, h, y = t["g"], t["u"], t["h"], t["y"]
    x_np = _np(x)

    # gate and up: the same (XH)_Q (quantized once, forward_shared)
    for lay, ctx, out, grad_in, gw, w in ((mlp.gate, mlp.ctx[0], g, t["dg"], gw_g, wg),
                                          (mlp.up, mlp.ctx[1], u, t["du"], gw_u, wu)):
        xq, sx, wq, sw = ctx.saved(lay)
        check_forward(orc, 0, x_np, _np(w), xq, sx, wq, sw, out)
        ops = ctx.error_operands(lay)
        ex_key = "ex_gate" if lay is mlp.gate else "ex_up"
        check_backward(orc, 0, _np(grad_in), xq, sx, wq, sw, ops, t[ex_key], gw)
    # down: input h, output y; its error is dy, its E_X is dh
    xq, sx, wq, sw = mlp.ctx[2].saved(mlp.down)
    check_forward(orc, 0, _np(h), _np(wd), xq, sx, wq, sw, y)
    ops = mlp.ctx[2].error_operands(mlp.down)
    check_backward(orc, 0, _np(dy), xq, sx, wq, sw, ops, t["dh"], gw_d)

    # glue: h = silu(g) u, (dg, du) = SwiGLU'(dh), dx = ex_gate + ex_up
    gf, uf, dhf = g.float(), u.float(), t["dh"].float()
    s = torch.sigmoid(gf)
    for got, ref in ((h, gf * s * uf), (t["du"], dhf * gf * s), (t["dg"], dhf * uf * s * (1 + gf * (1 - s)))):
        err = (got.float() - ref).abs()
        assert bool((err <= 2 ** -6 * ref.abs() + 1e-30).all())
    assert torch.equal(dx, (t["ex_gate"].float() + t["ex_up"].float()).to(bf))
    del check, lib


# ------------------------------------------------------------------ long K
# The INT8 GEMM accumulates in s32 TMEM, exact for K <= 133,144; the
# reference accumulates in int64 (quantize.hpp:358-371).  Longer
# contractions (the G GEMM over > 131072 tokens) are summed in int64 over K
# slices.  These cases overflow int32 on purpose.

def test_qmatmul_int8_long_k_exceeds_int32(H):
    K, M, N = 140000, 256, 128
    g = torch.Generator(device="cuda").manual_seed(9)
    a = torch.full((K, M), 127, dtype=torch.int8, device="cuda")            # MN-major [K][M]
    signs = torch.randint(0, 2, (K, N), generator=g, device="cuda", dtype=torch.int8) * 2 - 1
    b = torch.full((K, N), 127, dtype=torch.int8, device="cuda")
    b[:, 1::2] *= signs[:, 1::2]                                             # even columns: |acc| = K*127^2
    sa = torch.tensor([1.0 / 127], device="cuda")
    sb = torch.tensor([3.0 / 127], device="cuda")
    acc = a.t().double() @ b.double()
    assert float(acc.abs().max()) > 2 ** 31
    want = _epilogue(acc, sa, sb)
    got = H.qmatmul(a, b, sa, sb, a_kmajor=False, b_kmajor=False)
    assert torch.equal(got, want)
    got_bf = H.qmatmul(a, b, sa, sb, a_kmajor=False, b_kmajor=False, out="bf16")
    assert torch.equal(got_bf, want.to(torch.bfloat16))
    # fused right transform along N (the G path's transform_right_ht)
    got_r = H.qmatmul(a, b, sa, sb, a_kmajor=False, b_kmajor=False, had_block=128)
    want_r = H.transform_right(want.contiguous(), 128)
    assert torch.equal(got_r, want_r)
    # raw s32 accumulators cannot hold this product: rejected, not wrapped
    with pytest.raises(ValueError):
        H.qmatmul(a, b, sa, sb, a_kmajor=False, b_kmajor=False, out="s32")


def test_layer_grad_w_over_139264_tokens(H, orc):
    """HALO-2 INT8 backward whose G GEMM contracts 139264 tokens with every
    product at +127*127 on one column per block (|acc| ~ 2.25e9 > 2^31)."""
    b, m, n = 139264, 256, 256
    x = torch.ones(b, m, dtype=torch.bfloat16, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(3)
    w = (torch.randn(n, m, generator=g, device="cuda") / 16).to(torch.bfloat16)
    e = torch.full((b, n), 1e-3, device="cuda").to(torch.bfloat16)
    layer = H.HaloLinearLayer(w, H.halo2(0, BLOCK), out_dtype=torch.float32)
    ctx = H.SavedContext()
    y = layer.forward(x, ctx)
    back = layer.backward(ctx, e)
    ctx.check()
    xq, sx, wq, sw = ctx.saved(layer)
    ops = ctx.error_operands(layer)
    acc = _exact_acc(ops["eq"].t(), xq, 0)
    assert float(acc.abs().max()) > 2 ** 31
    del acc
    check_forward(orc, 0, _np(x), _np(w), xq, sx, wq, sw, y)
    check_backward(orc, 0, _np(e), xq, sx, wq, sw, ops, back.e_x, back.grad_w)
